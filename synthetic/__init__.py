"""Seeded synthetic input generators (no method arithmetic; see inputs.py)."""
from .inputs import *  # noqa: F401,F403
