# the round's GPU check: full suite, bench lines for every config, exact mode, ring vs pair on MC
set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/r_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/r_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/r_smoke.txt
timeout 300 python bench.py > gpurun_out/r_bench.json 2> gpurun_out/r_bench.err
timeout 300 python bench.py --config mc > gpurun_out/r_bench_mc.json 2> gpurun_out/r_bench_mc.err
FVB_KERNEL=ring timeout 300 python bench.py --config mc > gpurun_out/r_bench_mc_ring.json 2> gpurun_out/r_bench_mc_ring.err
timeout 300 python bench.py --config kh3d > gpurun_out/r_bench_kh3d.json 2> gpurun_out/r_bench_kh3d.err
timeout 300 python bench.py --config bqmc --steps 10 --no-cpu > gpurun_out/r_bench_bqmc.json 2> gpurun_out/r_bench_bqmc.err
FVB_BENCH_ARITH=exact timeout 300 python bench.py --no-cpu --e2e-reps 1 --steps 30 > gpurun_out/r_bench_exact.json 2> gpurun_out/r_bench_exact.err
timeout 600 python bench.py --impl reference > gpurun_out/r_bench_ref.json 2> gpurun_out/r_bench_ref.err
echo done
