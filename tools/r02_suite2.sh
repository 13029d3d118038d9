set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/s2_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/s2_tests.txt
echo done
