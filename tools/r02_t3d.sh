mkdir -p gpurun_out/t3d
timeout 1500 python -m pytest tests/test_gpu_benchsize.py -q -x > gpurun_out/t3d/benchsize.txt 2>&1; echo "rc=$?" >> gpurun_out/t3d/benchsize.txt
timeout 300 python bench.py --config kh3d --no-cpu > gpurun_out/t3d/kh3d.json 2>/dev/null
tail -n 3 gpurun_out/t3d/benchsize.txt
python -c "import json;d=json.loads(open('gpurun_out/t3d/kh3d.json').read().strip().splitlines()[-1]);print(d['value'], d['config']['parity'])"
