# A/B of a compile-time variant: default build vs ADJ_NVCC_EXTRA (rebuilds the kernels)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
DBGS=0 SWEEP="c2:1 c2:0 c3:2" bash tools/gpu_exp.sh; sed "s/^/A /" gpurun_out/exp.log > gpurun_out/ab.log
touch paper_2101_01025_b200/csrc/*.cu
ADJ_NVCC_EXTRA="$VARIANT" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
DBGS=0 SWEEP="c2:1 c2:0 c3:2" bash tools/gpu_exp.sh; sed "s/^/B /" gpurun_out/exp.log >> gpurun_out/ab.log
