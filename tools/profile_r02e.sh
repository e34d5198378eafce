# Round-2 closing evidence on the final tree (the GPU suite and smoke ran in tools/gpu_verify.sh):
# every config's bench line, the reference arm, the c3 launch list, ncu --set full of c3 / c4.
set -x
OUT=gpurun_out/prof8; mkdir -p $OUT
timeout 900 python bench.py > $OUT/bench_c3.log 2>&1
for c in c4 c2 c5 q5 c1 x131071; do timeout 600 python bench.py --config $c --steps ${STEPS:-10} > $OUT/bench_$c.log 2>&1; done
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_reference_c3.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_c3_bench.csv python bench.py --no-cpu --no-check --no-compare --steps 2 --warmup 3 --sustain-s 0 > $OUT/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'leafw_kernel|preadd2_kernel|combine_kernel' -c 4 -o /tmp/full_c3 -f python tools/run_one.py --config c3 --reps 1 --io16 > $OUT/ncu_full_c3.log 2>&1
python tools/ncu_summary.py /tmp/full_c3.ncu-rep > $OUT/ncu_full_c3_d2.json 2>&1
timeout 600 ncu --set full --clock-control none -k regex:'leafw_kernel|preadd2_kernel' -c 2 -o /tmp/full_c4 -f python tools/run_one.py --config c4 --reps 1 --io16 > $OUT/ncu_full_c4.log 2>&1
python tools/ncu_summary.py /tmp/full_c4.ncu-rep > $OUT/ncu_full_c4_d2.json 2>&1
du -sh $OUT
