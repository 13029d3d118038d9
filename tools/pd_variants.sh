# ring prefetch depth A/B: default (PD 2) vs -DFVB_RING_PD=1/3/4 variant builds
mkdir -p gpurun_out
for rep in 1 2; do
for v in main pd1 pd3 pd4; do
  if [ $v = main ]; then L=""; else L="$PWD/build/$v/libfvb200.so"; fi
  FVB_LIB=$L timeout 120 python bench.py --no-cpu --e2e-reps 1 --steps 30 > gpurun_out/pd_${v}_${rep}.json 2> gpurun_out/pd_${v}_${rep}.err
done; done
for v in pd1 pd3 pd4; do
  FVB_LIB=$PWD/build/$v/libfvb200.so timeout 300 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pd_parity_$v.log 2>&1
done
for v in main pd1 pd3 pd4; do
  if [ $v = main ]; then L=""; else L="$PWD/build/$v/libfvb200.so"; fi
  FVB_LIB=$L timeout 120 python bench.py --no-cpu --e2e-reps 1 --steps 10 --config mc > gpurun_out/pd_mc_$v.json 2>&1
  FVB_LIB=$L timeout 120 python bench.py --no-cpu --e2e-reps 1 --steps 10 --config bqmc > gpurun_out/pd_bq_$v.json 2>&1
done
