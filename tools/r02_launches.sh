# ncu launch list of the timed bench command (from the saved developed state, no warm-up march)
set -x
mkdir -p gpurun_out/final
python tools/make_state.py 1.0 /tmp/kh2d_t1.npy > /dev/null 2>&1
CMD="python bench.py --state-file /tmp/kh2d_t1.npy --warm-time 0 --steps 20 --warmup 5 --no-cpu --e2e-reps 1 --sustain 0.1"
timeout 300 $CMD > gpurun_out/final/launch_plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/final/launches_state.csv $CMD > gpurun_out/final/ncu_state.log 2>&1
gzip -f gpurun_out/final/launches_state.csv
echo done
