# pair kernel: parity + bench, then the ncu captures of every kernel
set -x
mkdir -p gpurun_out
FVB_KERNEL=pair python -m pytest tests/test_gpu_parity.py tests/test_gpu_benchsize.py tests/test_gpu_fullsize.py -x -q > gpurun_out/p2_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/p2_tests.txt
python -m pytest tests/test_gpu_numerics.py tests/test_gpu_parallel_dist.py tests/test_gpu_reference_suite.py tests/test_gpu_bench_contract.py -q > gpurun_out/f_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/f_tests.txt
for rep in 1 2; do
  timeout 200 python bench.py --no-cpu --e2e-reps 1 --steps 30 > gpurun_out/p2_ring_$rep.json 2> gpurun_out/p2_ring_$rep.err
  FVB_KERNEL=pair timeout 200 python bench.py --no-cpu --e2e-reps 1 --steps 30 > gpurun_out/p2_pair_$rep.json 2> gpurun_out/p2_pair_$rep.err
done
FVB_KERNEL=pair timeout 200 python bench.py --no-cpu --e2e-reps 1 --steps 10 --config mc > gpurun_out/p2_pair_mc.json 2> gpurun_out/p2_pair_mc.err
FVB_KERNEL=pair FVB_BENCH_ARITH=exact timeout 200 python bench.py --no-cpu --e2e-reps 1 --steps 30 > gpurun_out/p2_pair_exact.json 2> gpurun_out/p2_pair_exact.err
FVB_BENCH_ARITH=exact timeout 200 python bench.py --no-cpu --e2e-reps 1 --steps 30 > gpurun_out/p2_ring_exact.json 2> gpurun_out/p2_ring_exact.err
bash tools/r02_ncu_all.sh
