python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for dbg in ${DBGS:-0 2}; do echo "dbg=$dbg"; ADJ_LEAF_DEBUG=$dbg bash tools/sweep.sh ${SWEEP:-c2:0 c2:1}; done > gpurun_out/exp.log 2>&1
