# ring3i spill-free variant: parity + A/B bench (KH3D 512^3)
mkdir -p gpurun_out/r3a
FVB_LIB=build/r3a/libfvb200.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_benchsize.py tests/test_gpu_parallel.py tests/test_gpu_fused_halo.py -q -x > gpurun_out/r3a/tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r3a/tests.txt
for i in 1 2; do
  timeout 300 python bench.py --config kh3d --no-cpu > gpurun_out/r3a/base_$i.json 2>/dev/null
  FVB_LIB=build/r3a/libfvb200.so timeout 300 python bench.py --config kh3d --no-cpu > gpurun_out/r3a/r3a_$i.json 2>/dev/null
done
for f in gpurun_out/r3a/*.json; do echo $f $(python -c "import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print(d['value'], d['roofline']['frac'])" 2>&1 | tail -1); done
tail -n 2 gpurun_out/r3a/tests.txt
