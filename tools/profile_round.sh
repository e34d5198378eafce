# Round evidence: bench lines for every config, the ncu launch list of the default bench command,
# and one ncu --set full capture of each hot-path kernel (summarised by tools/ncu_summary.py).
set -x
OUT=gpurun_out/prof; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1
python bench.py > $OUT/bench_c2.log 2>&1
for c in c1 c3 c4 c5 q5 x131071; do python bench.py --config $c --steps ${STEPS:-10} > $OUT/bench_$c.log 2>&1; done
python bench.py --config c5 --herk alg1 --steps 10 --no-cpu > $OUT/bench_c5_herk_alg1.log 2>&1
python bench.py --config c2 --depth 0 --no-cpu --no-compare > $OUT/bench_c2_d0.log 2>&1
python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_reference_c2.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_c2_bench.csv python bench.py --no-cpu --no-check --steps 2 --warmup 3 --sustain-s 0 > $OUT/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'leaf2_kernel|preadd_kernel|combine_kernel' -s 3 -c 3 -o /tmp/full_c2_d1 -f python tools/run_one.py --config c2 --depth 1 --reps 2 --io16 > $OUT/ncu_full.log 2>&1
python tools/ncu_summary.py /tmp/full_c2_d1.ncu-rep > $OUT/ncu_full_c2_d1.json 2>&1
ncu --set full --clock-control none -k regex:'preadd_kernel|combine_kernel' -s 2 -c 2 -o /tmp/full_c2_d1_u32 -f python tools/run_one.py --config c2 --depth 1 --reps 2 > $OUT/ncu_full_u32.log 2>&1
python tools/ncu_summary.py /tmp/full_c2_d1_u32.ncu-rep > $OUT/ncu_full_c2_d1_u32.json 2>&1
ncu --set full --clock-control none -k regex:'leaf2_kernel|split_plain_kernel' -s 2 -c 2 -o /tmp/full_c2_d0 -f python tools/run_one.py --config c2 --depth 0 --reps 2 --io16 > $OUT/ncu_full_d0.log 2>&1
python tools/ncu_summary.py /tmp/full_c2_d0.ncu-rep > $OUT/ncu_full_c2_d0.json 2>&1
ncu --set full --clock-control none -k regex:'twom_kernel|split_kernel' -s 2 -c 2 -o /tmp/full_c5 -f python tools/run_one.py --config c5 --depth 0 --reps 2 > $OUT/ncu_full_c5.log 2>&1
python tools/ncu_summary.py /tmp/full_c5.ncu-rep > $OUT/ncu_full_c5_d0.json 2>&1
