# ring3i tile height A/B (8 rows / 2 blocks per SM vs 16 rows / 1 block per SM)
mkdir -p gpurun_out/nty
FVB_LIB=build/nty16/libfvb200.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_benchsize.py tests/test_gpu_ragged.py tests/test_gpu_parallel.py -q -x -k "3d or kh3d or ring3i or decomp" > gpurun_out/nty/tests.txt 2>&1; echo "rc=$?" >> gpurun_out/nty/tests.txt
for i in 1 2; do
  timeout 300 python bench.py --config kh3d --no-cpu > gpurun_out/nty/base_$i.json 2>/dev/null
  FVB_LIB=build/nty16/libfvb200.so timeout 300 python bench.py --config kh3d --no-cpu > gpurun_out/nty/var_$i.json 2>/dev/null
done
for f in gpurun_out/nty/*.json; do echo $f $(python -c "import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print(d['value'])" 2>&1 | tail -1); done
tail -n 2 gpurun_out/nty/tests.txt
