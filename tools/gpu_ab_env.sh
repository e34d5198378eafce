# A/B of a runtime switch: default vs with $ENVSET (e.g. ADJ_LEAF_STATIC=1), sweep $SWEEP twice
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for i in 1 2; do
DBGS=0 bash tools/gpu_exp.sh; sed "s/^/A /" gpurun_out/exp.log >> gpurun_out/ab.log
env $ENVSET DBGS=0 bash tools/gpu_exp.sh; sed "s/^/B /" gpurun_out/exp.log >> gpurun_out/ab.log
done
