# scratch GPU call used during round 2 (edited per call)
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
AB_WORKLOADS="SWEEP MIX TXT TINY" timeout 1200 bash tools/ab_run.sh gpurun_out/ab_modes.jsonl build_variants/cur/libsaturn.so build_variants/modes/libsaturn.so
tail -3 gpurun_out/ab_modes.jsonl.err
python - <<'PY'
import json
for l in open('gpurun_out/ab_modes.jsonl'):
    d=json.loads(l); print(d['lib'][:22], d['workload'], 'eval %.4g' % d['evaluate_plans_per_s'], 'step %.4f' % d['step_ms'], 'kga %.4f' % d['ga_kernel_ms'], d['best'])
PY
