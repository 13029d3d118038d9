# ncu evidence for every kernel (profiles/r02_ncu_*): plain run first, then --set full captures,
# exported to CSV on the box (raw metrics + per-line source) to stay under gpurun's 64 MiB return
set -x
mkdir -p gpurun_out/ncu
python tools/make_state.py 1.0 /tmp/kh2d_t1.npy > gpurun_out/n_state.log 2>&1
N="ncu --set full --clock-control none --import-source on"
for m in bqmc mc halo kh3d kh2d; do timeout 300 python tools/profile_kernels.py $m > gpurun_out/n_plain_$m.log 2>&1 || echo "plain $m failed"; done
cap() {  # name, regex, skip, count, mode
  timeout 900 $N -k regex:"$2" -s $3 -c $4 -o /tmp/$1 python tools/profile_kernels.py $5 > gpurun_out/ncu/$1.log 2>&1
  ncu -i /tmp/$1.ncu-rep --page raw --csv > gpurun_out/ncu/$1_raw.csv 2>/dev/null
  ncu -i /tmp/$1.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/ncu/$1_source.csv 2>/dev/null
  gzip -f gpurun_out/ncu/$1_source.csv
  rm -f /tmp/$1.ncu-rep
}
cap bqmc_ring "ring_kernel" 2 2 bqmc
cap bqmc_stats "moments_push|structure_pass" 3 3 bqmc
cap mc_init "init_eval|moments_push" 0 2 mc
cap halo "halo_instances" 2 2 halo
cap kh3d "ring3_kernel" 1 3 kh3d
cap kh2d "ring_kernel" 3 3 kh2d
FVB_KERNEL=pair cap kh2d_pair "pair_kernel" 3 3 kh2d
du -sh gpurun_out
echo done
