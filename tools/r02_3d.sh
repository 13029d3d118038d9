# 3D all-interior ring kernel: parity + bench vs the previous 3D kernel
set -x
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_benchsize.py tests/test_gpu_parallel.py tests/test_gpu_parallel_dist.py tests/test_gpu_fullsize.py -x -q > gpurun_out/t3_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/t3_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/t3_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/t3_smoke.txt
for rep in 1 2; do
  timeout 300 python bench.py --config kh3d --no-cpu > gpurun_out/t3_new_$rep.json 2> gpurun_out/t3_new_$rep.err
  FVB_KERNEL=ring3 timeout 300 python bench.py --config kh3d --no-cpu > gpurun_out/t3_old_$rep.json 2> gpurun_out/t3_old_$rep.err
done
timeout 300 python bench.py --config kh3d --no-cpu --cells 256 > gpurun_out/t3_new256.json 2> gpurun_out/t3_new256.err
FVB_BENCH_ARITH=exact timeout 300 python bench.py --config kh3d --no-cpu --cells 256 > gpurun_out/t3_new256_exact.json 2> gpurun_out/t3_new256_exact.err
python tools/profile_kernels.py kh3d > gpurun_out/t3_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ring3i -s 1 -c 3 -o /tmp/t3 python tools/profile_kernels.py kh3d > gpurun_out/t3_ncu.log 2>&1
mkdir -p gpurun_out/ncu
ncu -i /tmp/t3.ncu-rep --page raw --csv > gpurun_out/ncu/kh3d_i_raw.csv 2>/dev/null
ncu -i /tmp/t3.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null | gzip > gpurun_out/ncu/kh3d_i_source.csv.gz
echo done
