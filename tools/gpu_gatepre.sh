# Soft claim-wave gate: a gated job issues its first ADJ_LEAF_GATE_PRE stages before it waits
# (0 = the hard gate), c3 / c4 under the power cap, alternating; parity with it on
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
: > gpurun_out/gatepre.jsonl
for cfg in c3 c4; do for rep in 1 2; do for g in 0 2 4 8; do
  ADJ_LEAF_GATE_PRE=$g timeout 300 python tools/power_probe.py --config $cfg --seconds 5 --tag pre$g >> gpurun_out/gatepre.jsonl 2>>gpurun_out/gatepre.err
done; done; done
ADJ_LEAF_GATE_PRE=4 timeout 900 python -m pytest tests/test_gpu_fullsize_exact.py -x -q -m gpu -k "c3 or c4 or c2" > gpurun_out/gatepre_parity.log 2>&1; echo parity=$?
