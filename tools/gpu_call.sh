# scratch GPU call used during round 2 (edited per call)
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for w in TXT MIX SWEEP; do
  s="0 1 2"; [ $w != TXT ] && s=0
  timeout 300 python tools/quality_gpu.py --workload $w --seeds $s --bar profiles/r1/quality_bar$([ $w != TXT ] && echo _$w).json --out gpurun_out/quality_v5_$w.json | cut -c1-200
done
