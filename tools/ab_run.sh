# A/B of libsaturn builds on the GPU box: tools/ab_run.sh OUT LIB1 LIB2 ... (workloads: $AB_WORKLOADS or TXT MIX SWEEP)
out=$1; shift
for w in ${AB_WORKLOADS:-TXT MIX SWEEP}; do for lib in "$@"; do python tools/variant_bench.py $lib $w; done; done > $out 2> $out.err
