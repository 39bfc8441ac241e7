# scratch GPU call used during round 2 (edited per call)
timeout 900 python tools/pop_scaling.py TXT 2>&1 | tail -5
