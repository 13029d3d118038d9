set -x
mkdir -p gpurun_out
for rep in 1 2 3; do
  timeout 200 python bench.py --no-cpu --e2e-reps 1 --steps 30 > gpurun_out/o_main_$rep.json 2> gpurun_out/o_main_$rep.err
  FVB_LIB=$PWD/build/xopt/libfvb200.so timeout 200 python bench.py --no-cpu --e2e-reps 1 --steps 30 > gpurun_out/o_xopt_$rep.json 2> gpurun_out/o_xopt_$rep.err
done
echo done
