# fused two-level K1: parity tests
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_k1_fused.py tests/test_gpu_lowmem.py -q > gpurun_out/pytest_k1f.log 2>&1; echo pytest=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_all=$?
