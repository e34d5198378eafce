# k-block rotation (ADJ_KROT) A/B: GPU suite, back-to-back c3 / c4 / c2 probes, leaf DRAM bytes
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
O=gpurun_out/krot.log; : > $O
for c in c3 c4; do for r in 1 0 1 0; do ADJ_KROT=$r python tools/power_probe.py --config $c --tag ${c}_krot$r >> $O 2>&1; done; done
for r in 1 0 1 0; do ADJ_KROT=$r python tools/power_probe.py --config c2 --seconds 3 --tag c2_krot$r >> $O 2>&1; done
grep '^{' $O | cut -c1-200
for r in 1 0; do for c in c3 c2; do
ADJ_KROT=$r timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:leaf2_kernel -c 1 --csv python tools/run_one.py --config $c --reps 1 --io16 > gpurun_out/ncu_krot${r}_$c.csv 2>&1
grep -E "dram__bytes|hit_rate|duration" gpurun_out/ncu_krot${r}_$c.csv | awk -F'","' -v t="krot$r $c" '{print t, $(NF-2), $(NF-1), $NF}'
done; done
