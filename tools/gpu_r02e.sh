mkdir -p gpurun_out
VAR=IBGM_XFLAT VALS="2 3" CFGS="4" K4=60 bash tools/ab_env.sh 2>&1 | tee gpurun_out/ab_xflat.txt
IBGM_XFLAT=3 timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "config4" 2>&1 | tail -2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_(xwarp|strided|lines|spread|interp|force)" --launch-skip 9 -c 12 -o /tmp/r02d_full4 python tools/run_steps.py 4 3 > /tmp/r02d_full4.log 2>&1; echo ncu rc=$?
PROFILE_OUT=gpurun_out python tools/profile_summary.py r02d - /tmp/r02d_full4.ncu-rep 4 > /dev/null 2>&1; echo summ rc=$?
timeout 300 python tools/ncu_src_lines.py /tmp/r02d_full4.ncu-rep "k_xwarp<12, 0" 40 > gpurun_out/r02d_s1_lines.txt 2>&1
timeout 300 python tools/ncu_opcodes.py /tmp/r02d_full4.ncu-rep "k_xwarp<12, 0" 30 > gpurun_out/r02d_s1_opcodes.txt 2>&1
ncu -i /tmp/r02d_full4.ncu-rep --page details -k regex:"k_xwarp<12, 0" > gpurun_out/r02d_s1_details.txt 2>&1
ls -la gpurun_out
