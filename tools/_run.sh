for ap in 0 1; do for pv in 0 1 2; do PROBE_APPEND=$ap TM_POLY=$pv timeout 120 python tools/power_probe.py; done; done
