# dispatch-order balance of the pair kernel's chunk heights: parity + A/B over weights
mkdir -p gpurun_out/bal
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_benchsize.py tests/test_gpu_ragged.py -q -x > gpurun_out/bal/tests.txt 2>&1; echo "rc=$?" >> gpurun_out/bal/tests.txt
for i in 1 2; do
  for w in 0 default 1.05,1,0.95 1.15,1,0.87 1.12,1.0,0.88; do
    if [ $w = default ]; then unset FVB_PAIR_BALANCE; else export FVB_PAIR_BALANCE=$w; fi
    timeout 300 python bench.py --no-cpu --e2e-reps 1 --steps 50 > gpurun_out/bal/w_${w}_$i.json 2>/dev/null
  done
done
unset FVB_PAIR_BALANCE
FVB_LIB=build/bt/libfvb200.so python tools/block_times.py gpurun_out/bal/bt.json > /dev/null 2>&1
for f in gpurun_out/bal/w_*.json; do echo $f $(python -c "import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print(d['value'], d['clocks']['sm_mhz'])" 2>&1 | tail -1); done
tail -n 2 gpurun_out/bal/tests.txt
python -c "import json; d=json.load(open('gpurun_out/bal/bt.json')); print({k:(v['span_us'], v['block_us'], v['mean_block_over_span']) for k,v in d.items()})"
