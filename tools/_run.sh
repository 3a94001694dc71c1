for nl in 8 2 1; do for ap in 0 1; do SWEEP_NL=$nl SWEEP_APPEND=$ap timeout 120 python tools/sweep.py | sed "s/^/nl=$nl /"; done; done
