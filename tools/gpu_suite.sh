# full GPU suite + bench lines of c1 / c2 (quick) and the default (c3)
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 300 python bench.py --config c1 --steps 5 > gpurun_out/bench_c1.log 2>&1; echo bench_c1=$?
timeout 300 python bench.py --config c2 > gpurun_out/bench_c2.log 2>&1; echo bench_c2=$?
timeout 900 python bench.py > gpurun_out/bench_c3.log 2>&1; echo bench=$?
