# round-2 final evidence: GPU tests, bench line, ncu launch list, one --set full capture of a config-4 step
TAG=${TAG:-r02f} bash tools/gpu_check.sh
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_(xwarp|strided|lines|spread|interp|force)" --launch-skip 9 -c 12 -o /tmp/${TAG:-r02f}_full4 python tools/run_steps.py 4 3 > /tmp/${TAG:-r02f}_full4.log 2>&1; echo ncu rc=$?
PROFILE_OUT=gpurun_out python tools/profile_summary.py ${TAG:-r02f} - /tmp/${TAG:-r02f}_full4.ncu-rep 4 > /dev/null 2>&1; echo summ rc=$?
ls -la gpurun_out
