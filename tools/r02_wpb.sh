# pair kernel warps per block: parity with the variant libraries + A/B bench
mkdir -p gpurun_out/wpb
for v in wpb2 wpb4; do
  FVB_LIB=build/$v/libfvb200.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_benchsize.py -q -x > gpurun_out/wpb/tests_$v.txt 2>&1; echo "rc=$?" >> gpurun_out/wpb/tests_$v.txt
done
for i in 1 2; do
  timeout 300 python bench.py --no-cpu --e2e-reps 1 --steps 50 > gpurun_out/wpb/base_$i.json 2>/dev/null
  for v in wpb2 wpb4; do FVB_LIB=build/$v/libfvb200.so timeout 300 python bench.py --no-cpu --e2e-reps 1 --steps 50 > gpurun_out/wpb/${v}_$i.json 2>/dev/null; done
done
for v in wpb2 wpb4; do FVB_LIB=build/$v/libfvb200.so timeout 300 python bench.py --config mc --no-cpu > gpurun_out/wpb/mc_$v.json 2>/dev/null; done
for f in gpurun_out/wpb/*.json; do echo $f $(python -c "import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print(d['value'], d['roofline']['frac'])" 2>&1 | tail -1); done
tail -n 2 gpurun_out/wpb/tests_*.txt
