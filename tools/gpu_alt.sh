# K-direction alternation of the wide leaf's units (ADJ_LEAF_DEBUG 4096) and the scheme-2
# accumulator order hh, (hl + lh), ll (ADJ_ACC_ORDER=1) at c3 under the power cap; parity with both
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
: > gpurun_out/alt.jsonl
for rep in 1 2; do
  timeout 300 python tools/power_probe.py --config c3 --seconds 5 --tag base >> gpurun_out/alt.jsonl 2>>gpurun_out/alt.err
  ADJ_LEAF_DEBUG=4096 timeout 300 python tools/power_probe.py --config c3 --seconds 5 --tag alt >> gpurun_out/alt.jsonl 2>>gpurun_out/alt.err
  ADJ_ACC_ORDER=1 timeout 300 python tools/power_probe.py --config c3 --seconds 5 --tag order >> gpurun_out/alt.jsonl 2>>gpurun_out/alt.err
  ADJ_ACC_ORDER=1 ADJ_LEAF_DEBUG=4096 timeout 300 python tools/power_probe.py --config c3 --seconds 5 --tag order_alt >> gpurun_out/alt.jsonl 2>>gpurun_out/alt.err
done
ADJ_ACC_ORDER=1 ADJ_LEAF_DEBUG=4096 timeout 900 python -m pytest tests/test_gpu_fullsize_exact.py tests/test_gpu_parity.py -x -q -m gpu -k "c3 or 65521 or 40009 or vs_oracle" > gpurun_out/alt_parity.log 2>&1; echo parity=$?
