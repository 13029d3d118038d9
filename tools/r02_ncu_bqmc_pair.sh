# ncu of the Burgers pair kernel (bqmc shape: 4 instances x 2048^2, batched)
mkdir -p gpurun_out/nb
python tools/profile_kernels.py bqmc > gpurun_out/nb/plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pair_kernel -s 3 -c 3 -o /tmp/nb python tools/profile_kernels.py bqmc > gpurun_out/nb/ncu.log 2>&1
ncu -i /tmp/nb.ncu-rep --page raw --csv > gpurun_out/nb/bqmc_pair_raw.csv 2>/dev/null
ncu -i /tmp/nb.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null | gzip > gpurun_out/nb/bqmc_pair_source.csv.gz
tail -n 3 gpurun_out/nb/ncu.log
