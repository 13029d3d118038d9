for rep in 1 2; do
for v in main v96 v128; do
  if [ $v = main ]; then L=""; else L="$PWD/build/$v/libfvb200.so"; fi
  FVB_LIB=$L timeout 120 python bench.py --no-cpu --e2e-reps 1 --steps 30 > gpurun_out/nt_${v}_${rep}.json 2> gpurun_out/nt_${v}_${rep}.err
done; done
for v in v96 v128; do
  FVB_LIB=$PWD/build/$v/libfvb200.so timeout 300 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/nt_parity_$v.log 2>&1
  FVB_LIB=$PWD/build/$v/libfvb200.so timeout 120 python bench.py --no-cpu --e2e-reps 1 --steps 10 --config mc > gpurun_out/nt_mc_$v.json 2>&1
done
timeout 120 python bench.py --no-cpu --e2e-reps 1 --steps 10 --config mc > gpurun_out/nt_mc_main.json 2>&1
