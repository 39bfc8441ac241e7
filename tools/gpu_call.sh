set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 600 bash tools/ab_run.sh gpurun_out/ab_peel.jsonl build_variants/r1final/libsaturn.so paper_2309_01226_b200/libsaturn.so
cat gpurun_out/ab_peel.jsonl; tail -5 gpurun_out/ab_peel.jsonl.err
