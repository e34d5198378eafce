# quick re-check of a rebuilt library: smoke, the soak / race tests and the main parity file
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout -k 10 900 python -m pytest tests/test_gpu_soak.py tests/test_gpu_parity.py tests/test_abi.py -m gpu -x -q > gpurun_out/quick.log 2>&1; echo quick=$?
tail -3 gpurun_out/quick.log
