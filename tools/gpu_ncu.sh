python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
ADJ_LEAF_DEBUG=128 python tools/run_one.py --config c2 --depth 1 --reps 2 > gpurun_out/dbg_d1.log 2>&1
for d in ${DEPTHS:-1}; do
ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-leaf2_kernel} -s ${SKIP:-1} -c ${COUNT:-1} -o gpurun_out/ncu_c2_d$d -f python tools/run_one.py --config c2 --depth $d --reps 2 > gpurun_out/ncu_d$d.log 2>&1; echo ncu$d=$?
done
