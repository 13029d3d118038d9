mkdir -p gpurun_out
python tools/debug_fused.py kh2d64_weno2_50 > gpurun_out/dbg.txt 2>&1
echo done
