set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for d in 1 0; do
ncu --set full --clock-control none --import-source on -k regex:leaf2_kernel -s 1 -c 1 -o gpurun_out/leaf_c2_d$d -f python tools/run_one.py --config c2 --depth $d --reps 2 > gpurun_out/ncu_leaf_d$d.log 2>&1; echo ncu$d=$?
done
