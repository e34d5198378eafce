# Claim-wave gate of the wide leaf (ADJ_LEAF_GATE, diagnostics) at c3 / c4 under the power cap,
# alternating with the ungated default; then full-size exact parity at c3 with the gate on.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
: > gpurun_out/gate.jsonl
for cfg in ${CFGS:-c3 c4}; do for rep in 1 2; do for g in ${GATES:-0 50 80 95 100}; do
  ADJ_LEAF_GATE=$g timeout 300 python tools/power_probe.py --config $cfg --seconds 5 --tag gate$g >> gpurun_out/gate.jsonl 2>>gpurun_out/gate.err
done; done; done
ADJ_LEAF_GATE=${PGATE:-95} timeout 900 python -m pytest tests/test_gpu_fullsize_exact.py -x -q -m gpu -k "c3 or c4" > gpurun_out/gate_parity.log 2>&1; echo parity=$?
