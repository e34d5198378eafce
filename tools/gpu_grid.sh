# power-regime probes at c3 / c4: leaf grid capped (ADJ_LEAF_GRID) and half the operand stream
# (ADJ_LEAF_DEBUG=256: B operand not loaded, wrong result) -- is the capped step SM- or energy-bound?
O=gpurun_out/grid.log; : > $O
python tools/power_probe.py --config c3 --tag base >> $O 2>&1
ADJ_LEAF_GRID=132 python tools/power_probe.py --config c3 --tag grid132 >> $O 2>&1
ADJ_LEAF_GRID=116 python tools/power_probe.py --config c3 --tag grid116 >> $O 2>&1
ADJ_LEAF_GRID=100 python tools/power_probe.py --config c3 --tag grid100 >> $O 2>&1
ADJ_LEAF_DEBUG=256 python tools/power_probe.py --config c3 --tag skipb >> $O 2>&1
python tools/power_probe.py --config c3 --tag base2 >> $O 2>&1
python tools/power_probe.py --config c4 --tag c4 >> $O 2>&1
ADJ_LEAF_GRID=132 python tools/power_probe.py --config c4 --tag c4grid132 >> $O 2>&1
