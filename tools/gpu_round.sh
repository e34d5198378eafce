set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
python bench.py > gpurun_out/bench_c2.log 2>&1; echo bench=$?
bash tools/sweep.sh c2:0 c2:1 c2:2 c3:1 c3:2 c4:1 c5:1 c1:1 > gpurun_out/sweep.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv python bench.py --no-cpu --no-check --steps 2 --warmup 3 > gpurun_out/ncu_launch.log 2>&1; echo ncu=$?
