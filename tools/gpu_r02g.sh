# A/B of the lines per block (RI) of the strided psi passes after the cheaper reduced-system phase
mkdir -p gpurun_out
VAR=IBGM_RI_K3 VALS="16 8" CFGS="4" K4=100 bash tools/ab_env.sh 2>&1 | tee gpurun_out/ab_ri_k3.txt
VAR=IBGM_RI_K1 VALS="8 16" CFGS="4" K4=100 bash tools/ab_env.sh 2>&1 | tee gpurun_out/ab_ri_k1.txt
for v in 16 8; do echo "IBGM_RI_K3=$v"; IBGM_RI_K3=$v timeout 300 python tools/phase_bench.py 4; done 2>&1 | tee gpurun_out/r02g_phases.txt
