# scratch GPU call used during round 2 (edited per call)
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
AB_WORKLOADS="TXT MIX" timeout 600 bash tools/ab_run.sh gpurun_out/ab_prune.jsonl build_variants/v5/libsaturn.so paper_2309_01226_b200/libsaturn.so
python - <<'PY'
import json
for l in open('gpurun_out/ab_prune.jsonl'):
    d=json.loads(l); print(d['lib'][:22], d['workload'], 'eval %.4g' % d['evaluate_plans_per_s'], 'step %.4f' % d['step_ms'], 'kga %.4f' % d['ga_kernel_ms'])
PY
