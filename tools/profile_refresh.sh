set -x
mkdir -p gpurun_out
python tools/make_state.py 1.0 gpurun_out/kh2d_t1.npy > gpurun_out/state.log 2>&1
timeout 300 python bench.py > gpurun_out/r_bench.json 2> gpurun_out/r_bench.err
timeout 400 python bench.py --impl reference --steps 50 --warmup 5 > gpurun_out/r_bench_ref.json 2> gpurun_out/r_bench_ref.err
for bw in 6:1 8:1 10:1 12:1 16:1 8:2 8:3 16:2; do b=${bw%:*}; w=${bw#*:}
  FVB_BLOCKS_PER_SM=$b FVB_WAVES=$w timeout 120 python bench.py --no-cpu --e2e-reps 1 --steps 30 > gpurun_out/sweep_b${b}_w${w}.json 2>/dev/null
done
for h in 64 128 256; do FVB_MARCH_ROWS=$h timeout 120 python bench.py --no-cpu --e2e-reps 1 --steps 30 > gpurun_out/sweep_h${h}.json 2>/dev/null; done
timeout 120 python bench.py --no-cpu --e2e-reps 1 --steps 30 > gpurun_out/sweep_default.json 2>/dev/null
FVB_GRAPH_STEPS=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r_launches.csv python bench.py --state-file gpurun_out/kh2d_t1.npy --warm-time 0 --steps 10 --warmup 3 --no-cpu --e2e-reps 1 --sustain 0.1 > gpurun_out/r_ncu1.log 2>&1
FVB_GRAPH_STEPS=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:ring_kernel -s 6 -c 3 -o gpurun_out/r_ring_full python bench.py --state-file gpurun_out/kh2d_t1.npy --warm-time 0 --steps 3 --warmup 3 --no-cpu --e2e-reps 1 --sustain 0.1 > gpurun_out/r_ncu2.log 2>&1
rm -f gpurun_out/kh2d_t1.npy
