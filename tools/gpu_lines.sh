# the other configs' bench lines on the current build (10 steps each)
OUT=gpurun_out/lines; mkdir -p $OUT
for c in c4 c2 c5 q5 x131071; do timeout -k 10 400 python bench.py --config $c --steps 10 > $OUT/bench_$c.json 2>$OUT/bench_$c.err; echo $c=$?; done
