set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
python bench.py > gpurun_out/bench_default.log 2>&1; echo bench=$?
for d in 2 3; do python bench.py --config c3 --depth $d --no-cpu --no-compare --steps 10 > gpurun_out/bench_c3_d$d.log 2>&1; done
python bench.py --config c2 --depth 1 --no-cpu --no-compare > gpurun_out/bench_c2_d1.log 2>&1
python bench.py --config c2 --depth 0 --no-cpu --no-compare > gpurun_out/bench_c2_d0.log 2>&1
