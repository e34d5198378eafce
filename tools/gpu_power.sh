# power attribution at c3 under sw_power_cap (ADJ_LEAF_DEBUG switches) + the c3 launch list
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
O=gpurun_out/power.log; : > $O
python tools/power_probe.py --config c3 --tag base >> $O 2>&1
ADJ_LEAF_DEBUG=8 python tools/power_probe.py --config c3 --tag nomath >> $O 2>&1
ADJ_LEAF_DEBUG=2 python tools/power_probe.py --config c3 --tag noepi >> $O 2>&1
ADJ_LEAF_DEBUG=1 python tools/power_probe.py --config c3 --tag notma >> $O 2>&1
ADJ_LEAF_DEBUG=3 python tools/power_probe.py --config c3 --tag notma_noepi >> $O 2>&1
python tools/power_probe.py --config c3 --depth 3 --tag d3 >> $O 2>&1
python tools/power_probe.py --config c3 --tag base2 >> $O 2>&1
python tools/power_probe.py --config c4 --tag c4 >> $O 2>&1
python tools/power_probe.py --config c2 --tag c2 >> $O 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c3.csv python tools/run_one.py --config c3 --reps 1 --io16 > gpurun_out/ncu_c3.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c4.csv python tools/run_one.py --config c4 --reps 1 --io16 > gpurun_out/ncu_c4.log 2>&1
