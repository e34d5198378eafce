# ncu source-level capture of K1 (c3: scheme s8/u8, Y = i I; c4: K7, Rot2) and K4 (c3); reports
# stay in /tmp on the box, CSV exports come back
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in c3 c4; do
ncu --set full --clock-control none --import-source on -k regex:'preadd_kernel' -s 0 -c 2 -o /tmp/k1_$c -f python tools/run_one.py --config $c --reps 1 --io16 > gpurun_out/k1_$c.log 2>&1
ncu -i /tmp/k1_$c.ncu-rep --page raw --csv > gpurun_out/k1_${c}_raw.csv 2>&1
ncu -i /tmp/k1_$c.ncu-rep --page source --csv > gpurun_out/k1_${c}_source.csv 2>&1
python tools/ncu_summary.py /tmp/k1_$c.ncu-rep > gpurun_out/k1_${c}_summary.json 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:'combine_kernel' -s 0 -c 2 -o /tmp/k4_c3 -f python tools/run_one.py --config c3 --reps 1 --io16 > gpurun_out/k4_c3.log 2>&1
ncu -i /tmp/k4_c3.ncu-rep --page raw --csv > gpurun_out/k4_c3_raw.csv 2>&1
ncu -i /tmp/k4_c3.ncu-rep --page source --csv > gpurun_out/k4_c3_source.csv 2>&1
python tools/ncu_summary.py /tmp/k4_c3.ncu-rep > gpurun_out/k4_c3_summary.json 2>&1
du -sh gpurun_out
