# ncu of the round-2 default 2D/3D kernels + exact 3D old/new + alternate-kernel parity
set -x
mkdir -p gpurun_out/ncu
python -m pytest tests/test_gpu_parity.py -q -k alternate > gpurun_out/w_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/w_tests.txt
FVB_BENCH_ARITH=exact timeout 300 python bench.py --config kh3d --no-cpu --cells 256 > gpurun_out/w_exact3d_new.json 2> gpurun_out/w_exact3d_new.err
FVB_KERNEL=ring3 FVB_BENCH_ARITH=exact timeout 300 python bench.py --config kh3d --no-cpu --cells 256 > gpurun_out/w_exact3d_old.json 2> gpurun_out/w_exact3d_old.err
python tools/make_state.py 1.0 /tmp/kh2d_t1.npy > /dev/null 2>&1
N="ncu --set full --clock-control none --import-source on"
cap() {
  timeout 900 $N -k regex:"$2" -s $3 -c $4 -o /tmp/$1 python tools/profile_kernels.py $5 > gpurun_out/ncu/$1.log 2>&1
  ncu -i /tmp/$1.ncu-rep --page raw --csv > gpurun_out/ncu/$1_raw.csv 2>/dev/null
  ncu -i /tmp/$1.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null | gzip > gpurun_out/ncu/$1_source.csv.gz
  rm -f /tmp/$1.ncu-rep
}
python tools/profile_kernels.py kh2d > gpurun_out/w_plain2d.log 2>&1 && cap kh2d_pair "pair_kernel" 3 3 kh2d
python tools/profile_kernels.py kh3d > gpurun_out/w_plain3d.log 2>&1 && cap kh3d_i "ring3i" 1 3 kh3d
echo done
