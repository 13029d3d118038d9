# round-2 perf iteration on one B200: precision probe, GPU tests, bench sweep, ncu of the ring kernel
set -x
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mufu tools/mufu_precision.cu && /tmp/mufu > gpurun_out/p_mufu.txt 2>&1
python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/p_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/p_tests.txt
python tools/make_state.py 1.0 /tmp/kh2d_t1.npy > gpurun_out/p_state.log 2>&1
timeout 300 python bench.py --no-cpu > gpurun_out/p_bench.json 2> gpurun_out/p_bench.err
for b in 9 10; do FVB_BLOCKS_PER_SM=$b timeout 200 python bench.py --no-cpu --e2e-reps 1 --steps 30 > gpurun_out/p_bench_b$b.json 2>gpurun_out/p_bench_b$b.err; done
for c in mc bqmc kh3d; do timeout 300 python bench.py --no-cpu --config $c --steps 10 > gpurun_out/p_bench_$c.json 2>gpurun_out/p_bench_$c.err; done
FVB_GRAPH_STEPS=0 timeout 120 python bench.py --state-file /tmp/kh2d_t1.npy --warm-time 0 --steps 3 --warmup 3 --no-cpu --e2e-reps 1 --sustain 0.1 > gpurun_out/p_plain.log 2>&1 && \
FVB_GRAPH_STEPS=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:ring_kernel -s 6 -c 3 -o gpurun_out/p_ring_full python bench.py --state-file /tmp/kh2d_t1.npy --warm-time 0 --steps 3 --warmup 3 --no-cpu --e2e-reps 1 --sustain 0.1 > gpurun_out/p_ncu.log 2>&1
echo done
