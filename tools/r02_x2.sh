# interleaved pair physics (x2) vs sequential, register caps; 3D barrier change
set -x
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_benchsize.py -x -q > gpurun_out/x_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/x_tests.txt
for rep in 1 2; do
for v in main pairseq x2min11 x2min10; do
  L=""; [ $v != main ] && L="$PWD/build/$v/libfvb200.so"
  FVB_LIB=$L timeout 200 python bench.py --no-cpu --e2e-reps 1 --steps 30 > gpurun_out/x_${v}_$rep.json 2> gpurun_out/x_${v}_$rep.err
done; done
timeout 300 python bench.py --config kh3d --no-cpu > gpurun_out/x_kh3d.json 2> gpurun_out/x_kh3d.err
timeout 300 python bench.py --config kh3d --no-cpu --cells 256 > gpurun_out/x_kh3d256.json 2> gpurun_out/x_kh3d256.err
echo done
