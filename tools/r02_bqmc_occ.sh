# Burgers QMC: grid shaping at different resident-block assumptions
mkdir -p gpurun_out/bo
for b in default 16 20 24 28 32; do
  if [ $b = default ]; then unset FVB_BLOCKS_PER_SM; else export FVB_BLOCKS_PER_SM=$b; fi
  timeout 300 python bench.py --config bqmc --no-cpu > gpurun_out/bo/b_$b.json 2>/dev/null
done
unset FVB_BLOCKS_PER_SM
timeout 300 python bench.py --config bqmc --no-cpu > gpurun_out/bo/b_default2.json 2>/dev/null
for f in gpurun_out/bo/*.json; do echo $f $(python -c "import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print(d['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>&1 | tail -1); done
