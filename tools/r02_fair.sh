# per-SM progress balancing (FVB_FAIR) A/B on KH2D
mkdir -p gpurun_out/fair
FVB_LIB=build/fair400/libfvb200.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_benchsize.py -q -x > gpurun_out/fair/tests.txt 2>&1; echo "rc=$?" >> gpurun_out/fair/tests.txt
for i in 1 2; do
  timeout 300 python bench.py --no-cpu --e2e-reps 1 --steps 50 > gpurun_out/fair/base_$i.json 2>/dev/null
  for v in fair400 fair1500; do FVB_LIB=build/$v/libfvb200.so timeout 300 python bench.py --no-cpu --e2e-reps 1 --steps 50 > gpurun_out/fair/${v}_$i.json 2>/dev/null; done
done
for f in gpurun_out/fair/*.json; do echo $f $(python -c "import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print(d['value'], d['clocks']['sm_mhz'])" 2>&1 | tail -1); done
tail -n 2 gpurun_out/fair/tests.txt
