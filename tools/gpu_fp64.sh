mkdir -p gpurun_out
for i in 1 2 3; do tools/fp64_micro; done | tee gpurun_out/fp64_micro.jsonl
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed.sum,lts__t_bytes.sum
timeout 900 ncu --metrics $M --clock-control none -k regex:"k_(xwarp|strided|lines|spread|interp|force)" --launch-skip 9 -c 9 --csv python tools/run_steps.py 4 3 > gpurun_out/fp64_ncu4.csv 2> gpurun_out/fp64_ncu4.err; echo ncu4 rc=$?
timeout 900 ncu --metrics $M --clock-control none -k regex:"k_(xwarp|strided|lines|spread|interp|force)" --launch-skip 9 -c 9 --csv python tools/run_steps.py 3 3 > gpurun_out/fp64_ncu3.csv 2> gpurun_out/fp64_ncu3.err; echo ncu3 rc=$?
