python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for d in 1 0; do
ADJ_LEAF_DEBUG=16384 python tools/run_one.py --config c2 --depth $d --reps 2 > gpurun_out/exit_d$d.log 2>&1
done
