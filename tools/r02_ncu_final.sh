# refresh the ncu evidence of the default kernels with the final build:
# kh2d pair (bench state), mc (batched pair + batched moments + init), kh3d ring3i (512^3),
# plus the launch list of the timed bench command
set -x
mkdir -p gpurun_out/ncuf gpurun_out/ncuf_launch
python tools/make_state.py 1.0 /tmp/kh2d_t1.npy > gpurun_out/ncuf/state.log 2>&1
N="ncu --set full --clock-control none --import-source on"
for m in mc kh3d kh2d; do timeout 300 python tools/profile_kernels.py $m > gpurun_out/ncuf/plain_$m.log 2>&1 || echo "plain $m failed"; done
cap() {  # name, regex, skip, count, mode
  timeout 1200 $N -k regex:"$2" -s $3 -c $4 -o /tmp/$1 python tools/profile_kernels.py $5 > gpurun_out/ncuf/$1.log 2>&1
  ncu -i /tmp/$1.ncu-rep --page raw --csv > gpurun_out/ncuf/$1_raw.csv 2>/dev/null
  ncu -i /tmp/$1.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null | gzip > gpurun_out/ncuf/$1_source.csv.gz
  rm -f /tmp/$1.ncu-rep
}
cap kh2d_pair "pair_kernel" 3 3 kh2d
cap mc_pair "pair_kernel|moments_push|init_eval" 0 5 mc
cap kh3d_i "ring3i_kernel" 1 3 kh3d
CMD="python bench.py --state-file /tmp/kh2d_t1.npy --warm-time 0 --steps 20 --warmup 5 --no-cpu --e2e-reps 1 --sustain 0.1"
timeout 300 $CMD > gpurun_out/ncuf_launch/launch_plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/ncuf_launch/launches.csv $CMD > gpurun_out/ncuf_launch/ncu.log 2>&1
gzip -f gpurun_out/ncuf_launch/launches.csv
du -sh gpurun_out/ncuf
echo done
