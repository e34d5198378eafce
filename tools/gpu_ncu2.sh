python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
ncu --set full --clock-control none -k regex:preadd_kernel -s 2 -c 2 -o gpurun_out/ncu_c4_pre -f python tools/run_one.py --config c4 --depth 2 --reps 2 > gpurun_out/ncu_c4.log 2>&1; echo ncu=$?
python tools/ncu_summary.py gpurun_out/ncu_c4_pre.ncu-rep > gpurun_out/ncu_c4_pre.json
