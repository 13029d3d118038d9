# end-of-round evidence (second pass): GPU suite, smoke, bench lines, reference arm, ncu of the batched moments kernel
set -x
mkdir -p gpurun_out/final6/ncu
python -m pytest tests -m gpu -q > gpurun_out/final6/tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/final6/tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final6/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/final6/smoke.txt
for c in kh2d mc kh3d bqmc; do timeout 300 python bench.py --config $c > gpurun_out/final6/bench_$c.json 2> gpurun_out/final6/bench_$c.err; done
timeout 300 python bench.py --config kh3d --cells 1024 --steps 5 --e2e-steps 2 > gpurun_out/final6/bench_kh3d1024.json 2> gpurun_out/final6/bench_kh3d1024.err
FVB_BENCH_ARITH=exact timeout 300 python bench.py --no-cpu > gpurun_out/final6/bench_exact.json 2> gpurun_out/final6/bench_exact.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/final6/bench_ref.json 2> gpurun_out/final6/bench_ref.err



echo done
