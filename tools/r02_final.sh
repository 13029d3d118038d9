# end-of-round evidence on one B200: full GPU suite, smoke, bench lines (every config), reference arm, launch list
set -x
mkdir -p gpurun_out/final
python -m pytest tests -m gpu -q > gpurun_out/final/tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/final/tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/final/smoke.txt
timeout 300 python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err
timeout 300 python bench.py --config mc > gpurun_out/final/bench_mc.json 2> gpurun_out/final/bench_mc.err
timeout 300 python bench.py --config kh3d > gpurun_out/final/bench_kh3d.json 2> gpurun_out/final/bench_kh3d.err
timeout 300 python bench.py --config bqmc --steps 10 > gpurun_out/final/bench_bqmc.json 2> gpurun_out/final/bench_bqmc.err
FVB_BENCH_ARITH=exact timeout 300 python bench.py --no-cpu > gpurun_out/final/bench_exact.json 2> gpurun_out/final/bench_exact.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/final/bench_ref.json 2> gpurun_out/final/bench_ref.err
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/final/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/final/launches.csv python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/final/ncu.log 2>&1
gzip -f gpurun_out/final/launches.csv
echo done
