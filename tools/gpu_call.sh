# scratch GPU call used during round 2 (edited per call)
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
