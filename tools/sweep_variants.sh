#!/bin/bash
# Tuning sweep run ON the GPU box: rebuilds the library with -D variants and times the affected
# streaming cases (graph-timed, tools/streambench.py).  Usage: tools/sweep_variants.sh "case names" "flags A" "flags B" ...
cases="$1"; shift
for flags in "$@"; do
  echo "=== $flags"
  ML_NVCC_EXTRA="$flags" python -m paper_2501_14807_b200.build --force > /dev/null 2> gpurun_out/sweep_build.err || { tail -5 gpurun_out/sweep_build.err; continue; }
  python tools/streambench.py $cases 2>&1 | grep -E "ms "
done
python -m paper_2501_14807_b200.build --force > /dev/null
