set -x
mkdir -p gpurun_out
python -m pytest tests/test_gpu_fused_halo.py -q > gpurun_out/fh_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/fh_tests.txt
echo done
