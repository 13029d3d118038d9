set -x
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -x -q -k alternate > gpurun_out/sp_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/sp_tests.txt
for rep in 1 2; do
  timeout 200 python bench.py --config bqmc --steps 10 --no-cpu > gpurun_out/sp_ring_$rep.json 2> gpurun_out/sp_ring_$rep.err
  FVB_KERNEL=pair timeout 200 python bench.py --config bqmc --steps 10 --no-cpu > gpurun_out/sp_pair_$rep.json 2> gpurun_out/sp_pair_$rep.err
done
echo done
