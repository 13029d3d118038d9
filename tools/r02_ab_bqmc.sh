# A/B on the Burgers QMC bench: variant library $1 vs the in-tree build
v=$1
mkdir -p gpurun_out/abq_$v
for i in 1 2; do
  timeout 300 python bench.py --config bqmc --no-cpu > gpurun_out/abq_$v/base_$i.json 2>/dev/null
  FVB_LIB=build/$v/libfvb200.so timeout 300 python bench.py --config bqmc --no-cpu > gpurun_out/abq_$v/var_$i.json 2>/dev/null
done
for f in gpurun_out/abq_$v/*.json; do echo $f $(python -c "import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print(d['value'], d['roofline']['frac'], d['clocks'])" 2>&1 | tail -1); done
