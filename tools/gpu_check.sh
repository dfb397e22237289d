set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG:-r02d}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG:-r02d}_pytest.log
timeout 900 python bench.py > gpurun_out/${TAG:-r02d}_bench.json 2> gpurun_out/${TAG:-r02d}_bench.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG:-r02d}_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-extra > gpurun_out/${TAG:-r02d}_ncu.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/${TAG:-r02d}_pytest.log
