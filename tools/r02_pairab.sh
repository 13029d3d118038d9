# pair-kernel register caps vs the ring kernel (tools/variant.py builds)
set -x
mkdir -p gpurun_out
FVB_KERNEL=pair python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/q_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/q_tests.txt
FVB_KERNEL=pair FVB_LIB=$PWD/build/pairmin12/libfvb200.so python -m pytest tests/test_gpu_parity.py -x -q -k "kh2d or residual" > gpurun_out/q_tests12.txt 2>&1; echo "tests rc=$?" >> gpurun_out/q_tests12.txt
for rep in 1 2; do
for v in ring pair pairmin11 pairmin12 pairmin14 ringmin9; do
  L=""; K=""
  case $v in pair*) K=pair;; esac
  case $v in pairmin*|ringmin*) L="$PWD/build/$v/libfvb200.so";; esac
  FVB_KERNEL=$K FVB_LIB=$L timeout 200 python bench.py --no-cpu --e2e-reps 1 --steps 30 > gpurun_out/q_${v}_$rep.json 2> gpurun_out/q_${v}_$rep.err
done; done
echo done
