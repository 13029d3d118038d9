# A/B: variant library $1 vs the in-tree build (parity + KH2D / MC bench)
v=$1
mkdir -p gpurun_out/ab_$v
FVB_LIB=build/$v/libfvb200.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_benchsize.py tests/test_gpu_numerics.py -q -x > gpurun_out/ab_$v/tests.txt 2>&1; echo "rc=$?" >> gpurun_out/ab_$v/tests.txt
for i in 1 2; do
  timeout 300 python bench.py --no-cpu --e2e-reps 1 --steps 50 > gpurun_out/ab_$v/base_$i.json 2>/dev/null
  FVB_LIB=build/$v/libfvb200.so timeout 300 python bench.py --no-cpu --e2e-reps 1 --steps 50 > gpurun_out/ab_$v/var_$i.json 2>/dev/null
done
FVB_LIB=build/$v/libfvb200.so timeout 300 python bench.py --config mc --no-cpu > gpurun_out/ab_$v/var_mc.json 2>/dev/null
FVB_LIB=build/$v/libfvb200.so timeout 300 python bench.py --config bqmc --no-cpu > gpurun_out/ab_$v/var_bqmc.json 2>/dev/null
for f in gpurun_out/ab_$v/*.json; do echo $f $(python -c "import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print(d['value'], d['roofline']['frac'])" 2>&1 | tail -1); done
tail -n 2 gpurun_out/ab_$v/tests.txt
