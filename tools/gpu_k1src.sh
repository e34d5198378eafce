# ncu source-level capture of the fused K1 at c3 and c4 (CSV exports only)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in c3 c4; do
timeout 300 ncu --set full --clock-control none --import-source on -k regex:'preadd2_kernel' -c 1 -o /tmp/k1f_$c -f python tools/run_one.py --config $c --reps 1 --io16 > gpurun_out/k1f_$c.log 2>&1
ncu -i /tmp/k1f_$c.ncu-rep --page source --csv > gpurun_out/k1f_${c}_source.csv 2>&1
python tools/ncu_summary.py /tmp/k1f_$c.ncu-rep > gpurun_out/k1f_${c}_summary.json 2>&1
done
