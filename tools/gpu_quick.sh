# quick look: per-phase times and graph ms/step of config 4, then a parity subset
mkdir -p gpurun_out
timeout 300 python tools/phase_bench.py 4 2>&1 | tee gpurun_out/quick_phases.txt
timeout 300 python tools/ab_step.py 4 100 2>&1 | tee -a gpurun_out/quick_phases.txt
timeout 300 python tools/ab_step.py 3 400 2>&1 | tee -a gpurun_out/quick_phases.txt
