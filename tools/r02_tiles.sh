# tile dependency flags: parity + A/B bench
mkdir -p gpurun_out/tf
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_benchsize.py tests/test_gpu_uq.py tests/test_gpu_fullsize.py -q -x > gpurun_out/tf/tests.txt 2>&1; echo "rc=$?" >> gpurun_out/tf/tests.txt
for i in 1 2; do
  FVB_TILE_FLAGS=0 timeout 300 python bench.py --no-cpu --e2e-reps 1 --steps 50 > gpurun_out/tf/off_$i.json 2>gpurun_out/tf/off_$i.err
  timeout 300 python bench.py --no-cpu --e2e-reps 1 --steps 50 > gpurun_out/tf/on_$i.json 2>gpurun_out/tf/on_$i.err
done
timeout 300 python bench.py --config mc --no-cpu > gpurun_out/tf/mc_on.json 2>gpurun_out/tf/mc_on.err
timeout 300 python bench.py --config bqmc --no-cpu > gpurun_out/tf/bqmc_on.json 2>gpurun_out/tf/bqmc_on.err
for f in gpurun_out/tf/*.json; do echo $f $(python -c "import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print(d['value'], d['roofline']['frac'])" 2>&1 | tail -1); done
tail -2 gpurun_out/tf/tests.txt
