# ring register cap A/B: default (8 blocks/SM, <=128 regs) vs -DFVB_RING_MINB=9/10 (~94 regs) at 9/10 blocks/SM
mkdir -p gpurun_out
for rep in 1 2; do
  timeout 120 python bench.py --no-cpu --e2e-reps 1 --steps 30 > gpurun_out/mb_main_$rep.json 2>/dev/null
  for v in 9 10; do
    FVB_LIB=$PWD/build/mb$v/libfvb200.so FVB_BLOCKS_PER_SM=$v timeout 120 python bench.py --no-cpu --e2e-reps 1 --steps 30 > gpurun_out/mb_${v}_$rep.json 2>/dev/null
  done
  FVB_LIB=$PWD/build/mb10/libfvb200.so FVB_BLOCKS_PER_SM=8 timeout 120 python bench.py --no-cpu --e2e-reps 1 --steps 30 > gpurun_out/mb_10at8_$rep.json 2>/dev/null
done
