# A/B of the strided passes' reduced-system phase (IBGM_MFWARP: 0 = round-2d code path,
# 1 = mean-correction sums by warp partials, 2 = + register-tiled dense circulant S^-1)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "line_solve or config4 or ten_step" 2>&1 | tail -3 | tee gpurun_out/r02f_parity.txt
for v in 0 1 2; do echo "IBGM_MFWARP=$v"; IBGM_MFWARP=$v timeout 300 python tools/phase_bench.py 4; done 2>&1 | tee gpurun_out/r02f_phases.txt
VAR=IBGM_MFWARP VALS="0 1 2" CFGS="4 3 2" K4=100 bash tools/ab_env.sh 2>&1 | tee gpurun_out/ab_mfwarp.txt
