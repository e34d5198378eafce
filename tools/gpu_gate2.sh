# Claim-wave gate in the 256 x 256 leaf (leaf2_kernel): GPU suite, c3 forced onto leaf2
# (ADJ_LEAF_WIDE=0) with and without the gate, and the per-rank output-tile shares at c3 size.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
: > gpurun_out/gate2.jsonl
for rep in 1 2; do for g in 0 1100; do
  ADJ_LEAF_WIDE=0 ADJ_LEAF_GATE=$g timeout 300 python tools/power_probe.py --config c3 --seconds 5 --tag leaf2_gate$g >> gpurun_out/gate2.jsonl 2>>gpurun_out/gate2.err
done; done
for g in 0 1100; do
  echo "gate $g" >> gpurun_out/shard_gate.txt
  ADJ_LEAF_GATE=$g N=32768 P=65521 DEPTHS=1 GS="1 2 4 8" timeout 600 python tools/shard_time.py >> gpurun_out/shard_gate.txt 2>&1
done
