"""Pin strength: plausible mistakes in the oracle must fail a pin.

Each mutant is a one-line edit of oracle/tm_oracle.c (a dropped term, a
wrong sign, a missing scale, a wrong index, a missing normalisation),
compiled to a temporary library and run against tests/test_oracle_pins.py
through the TM_ORACLE_LIB override.  The pins must FAIL for every mutant.
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "tm_oracle.c")

MUTANTS = {
    "drop_previous_chunk": ("if (t - 1 > 0) out[n++] = t - 1;", ""),
    "drop_reference_chunk": ("out[n++] = 0;                       /* c_0", "/* c_0"),
    "no_softmax_scale": ("s[j] = dot * scale;", "s[j] = dot;"),
    "no_normalisation": ("double w = s[j] / l;", "double w = s[j];"),
    "euler_sign": ("out[i] = x[i] + dt * v[i];", "out[i] = x[i] - dt * v[i];"),
    "head_index": ("kr[j] = K + j * row + (int64_t)h * d;", "kr[j] = K + j * row;"),
    "interp_swapped": ("out[i] = t * x1[i] + (1.0 - t) * x0[i];", "out[i] = t * x0[i] + (1.0 - t) * x1[i];"),
    "prev_segment_dropped": ("if (Lp) { memcpy(K + Lr * row", "if (0) { memcpy(K + Lr * row"),
    "audio_window_unclamped": ("if (g < 0) g = 0;", "if (g < 0) g = -g;"),
    "audio_window_offset": ("int64_t g = f - window / 2 + i;", "int64_t g = f - window / 2 + i + 1;"),
    "sampler_no_time_factor": ("x[i] + (1.0 - t_cur) * u[i]", "x[i] + u[i]"),
    "sampler_renoise_swapped": ("t_next * x1_hat + (1.0 - t_next) * eps[i]",
                                "(1.0 - t_next) * x1_hat + t_next * eps[i]"),
}


@pytest.mark.parametrize("name", sorted(MUTANTS))
def test_mutant_is_caught(name, tmp_path):
    old, new = MUTANTS[name]
    src = open(SRC).read()
    assert src.count(old) == 1, f"mutation site for {name} not found exactly once"
    mut = tmp_path / "mutant.c"
    mut.write_text(src.replace(old, new))
    so = tmp_path / "libmutant.so"
    subprocess.check_call(["gcc", "-O1", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                           "-o", str(so), str(mut), "-lm"])
    env = dict(os.environ, TM_ORACLE_LIB=str(so), OMP_NUM_THREADS="4")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_oracle_pins.py")],
                       env=env, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode != 0, f"mutant {name} survived the pins:\n{r.stdout[-2000:]}"
