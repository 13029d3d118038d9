# pair kernel march length / waves sweep (KH2D 1024^2 fast)
mkdir -p gpurun_out/hs
for h in default 4 6 8 12 16 24; do
  if [ $h = default ]; then unset FVB_MARCH_ROWS; else export FVB_MARCH_ROWS=$h; fi
  timeout 200 python bench.py --no-cpu --e2e-reps 1 --steps 30 > gpurun_out/hs/h_$h.json 2>/dev/null
done
unset FVB_MARCH_ROWS
for w in 2 3 4; do FVB_WAVES=$w timeout 200 python bench.py --no-cpu --e2e-reps 1 --steps 30 > gpurun_out/hs/w_$w.json 2>/dev/null; done
for f in gpurun_out/hs/*.json; do echo $f $(python -c "import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print(d['value'])"); done
