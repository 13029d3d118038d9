# honest A/B (build/base = HEAD, build/var = working tree) on KH2D and the Burgers QMC config
tag=$1
mkdir -p gpurun_out/ab3_$tag
FVB_LIB=build/var/libfvb200.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_benchsize.py tests/test_gpu_ragged.py tests/test_gpu_uq.py -q -x > gpurun_out/ab3_$tag/tests.txt 2>&1; echo "rc=$?" >> gpurun_out/ab3_$tag/tests.txt
for i in 1 2 3; do
  for v in base var; do
    FVB_LIB=build/$v/libfvb200.so timeout 300 python bench.py --no-cpu --e2e-reps 1 --steps 50 > gpurun_out/ab3_$tag/kh2d_${v}_$i.json 2>/dev/null
    FVB_LIB=build/$v/libfvb200.so timeout 300 python bench.py --config bqmc --no-cpu > gpurun_out/ab3_$tag/bqmc_${v}_$i.json 2>/dev/null
  done
done
for f in gpurun_out/ab3_$tag/*.json; do echo $f $(python -c "import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print(d['value'], d['clocks']['sm_mhz'])" 2>&1 | tail -1); done
tail -n 2 gpurun_out/ab3_$tag/tests.txt
