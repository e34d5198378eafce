# L2 cache policies of the gated wide leaf's operand loads (ADJ_LEAF_DEBUG 4096: A evict_last,
# 8192: B evict_first) at c3 / c4 under the power cap, alternating with the default
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
: > gpurun_out/hint2.jsonl
for cfg in c3 c4; do for rep in 1 2; do for d in 0 4096 8192 12288; do
  ADJ_LEAF_DEBUG=$d timeout 300 python tools/power_probe.py --config $cfg --seconds 5 --tag hint$d >> gpurun_out/hint2.jsonl 2>>gpurun_out/hint2.err
done; done; done
