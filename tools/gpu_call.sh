# scratch GPU call used during round 2 (edited per call)
set -x
sed -i 's/population=1 << 22/population=1 << 23/' tools/variant_bench.py
AB_WORKLOADS="SWEEP" timeout 1800 bash tools/ab_run.sh gpurun_out/ab_nkl.jsonl build_variants/cur/libsaturn.so build_variants/nonkl/libsaturn.so build_variants/cur/libsaturn.so build_variants/nonkl/libsaturn.so
python - <<'PY'
import json
for f in ['gpurun_out/ab_nkl.jsonl']:
  for l in open(f):
    d=json.loads(l); print(d['lib'][-22:], d['workload'], 'eval %.4g' % d['evaluate_plans_per_s'], 'step %.4f' % d['step_ms'], 'kga %.4f' % d['ga_kernel_ms'], d['best'])
PY
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_nkl.txt 2>&1; echo pytest=$?; tail -2 gpurun_out/gputest_nkl.txt
