# K4 with 64 x 64 tile pairs of 256 threads (ADJ_K4_T64) against 32 x 32 / 64 threads, c3 / c4
# under the power cap; parity of the T = 64 instance
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
: > gpurun_out/k4t64.jsonl
for cfg in c3 c4; do for rep in 1 2; do
  timeout 300 python tools/power_probe.py --config $cfg --seconds 5 --tag t32 >> gpurun_out/k4t64.jsonl 2>>gpurun_out/k4t64.err
  ADJ_K4_T64=1 timeout 300 python tools/power_probe.py --config $cfg --seconds 5 --tag t64 >> gpurun_out/k4t64.jsonl 2>>gpurun_out/k4t64.err
done; done
ADJ_K4_T64=1 timeout 900 python -m pytest tests/test_gpu_fullsize_exact.py tests/test_gpu_parity.py -x -q -m gpu -k "c3 or c4 or vs_oracle or depth" > gpurun_out/k4t64_parity.log 2>&1; echo parity=$?
