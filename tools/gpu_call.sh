# scratch GPU call used during round 2 (edited per call)
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
AB_WORKLOADS="SWEEP TXT" timeout 900 bash tools/ab_run.sh gpurun_out/ab_gs.jsonl build_variants/prev/libsaturn.so build_variants/gs/libsaturn.so
tail -3 gpurun_out/ab_gs.jsonl.err
python - <<'PY'
import json
for l in open('gpurun_out/ab_gs.jsonl'):
    d=json.loads(l); print(d['lib'][:22], d['workload'], 'eval %.4g' % d['evaluate_plans_per_s'], 'step %.4f' % d['step_ms'], 'kga %.4f' % d['ga_kernel_ms'], d['best'])
PY
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_ga --launch-skip 20 --launch-count 1 \
  -o gpurun_out/prof_ga_txt_gs python bench.py --steps 2 --warmup 1 --no-cpu-baseline --kernel-only-n 0 > /dev/null 2>&1
