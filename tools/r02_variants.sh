# A/B of ring-kernel build variants (tools/variant.py) on one B200
set -x
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_benchsize.py -x -q > gpurun_out/v_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/v_tests.txt
for rep in 1 2; do
for v in main minb10 minb11 noskip minb10_noskip noxshfl; do
  if [ $v = main ]; then L=""; else L="$PWD/build/$v/libfvb200.so"; fi
  FVB_LIB=$L timeout 120 python bench.py --no-cpu --e2e-reps 1 --steps 30 > gpurun_out/v_${v}_${rep}.json 2> gpurun_out/v_${v}_${rep}.err
done; done
FVB_BLOCKS_PER_SM=8 timeout 120 python bench.py --no-cpu --e2e-reps 1 --steps 30 > gpurun_out/v_main_b8.json 2> gpurun_out/v_main_b8.err
for v in minb10 minb11; do
  FVB_LIB=$PWD/build/$v/libfvb200.so timeout 120 python bench.py --no-cpu --e2e-reps 1 --steps 10 --config mc > gpurun_out/v_mc_$v.json 2>&1
  FVB_LIB=$PWD/build/$v/libfvb200.so timeout 120 python bench.py --no-cpu --e2e-reps 1 --steps 10 --config bqmc > gpurun_out/v_bqmc_$v.json 2>&1
done
timeout 120 python bench.py --no-cpu --e2e-reps 1 --steps 10 --config mc > gpurun_out/v_mc_main.json 2>&1
timeout 120 python bench.py --no-cpu --e2e-reps 1 --steps 10 --config bqmc > gpurun_out/v_bqmc_main.json 2>&1
echo done
