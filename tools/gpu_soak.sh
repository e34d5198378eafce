# the repetition / two-stream race tests alone, timed
timeout -k 10 300 python -m pytest tests/test_gpu_soak.py -m gpu -x -q --durations=10 > gpurun_out/soak.log 2>&1; echo soak=$?
tail -25 gpurun_out/soak.log
