for flags in "-DML_CHAIN_LAZY_MINB=2" "-DML_CHAIN_LAZY_MINB=3"; do
  echo "=== $flags"
  ML_NVCC_EXTRA="$flags" python -m paper_2501_14807_b200.build --force > /dev/null 2> gpurun_out/sweep_build.err || { tail -5 gpurun_out/sweep_build.err; continue; }
  cuobjdump -res-usage paper_2501_14807_b200/libmeshlayers_b200.so 2>/dev/null | grep -A1 "chain_lazy_kernelILi1" | tail -1
  python bench.py --steps 300 --no-cpu --host-plane-reps 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['config']['stage_results']['chain']['ms'])"
done
