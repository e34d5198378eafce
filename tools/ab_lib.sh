# Dev tool: A/B of the in-tree library against $LIBB (another build) on bench config $CFG, alternating
# (the product binding loads only the in-tree libadjprod.so, so the two builds are swapped into place)
CFG=${CFG:-c2}; STEPS=${STEPS:-20}
L=paper_2101_01025_b200/libadjprod.so; cp $L /tmp/libA.so
for i in 1 2 3; do
cp /tmp/libA.so $L; python bench.py --config $CFG --no-cpu --no-check --no-compare --sustain-s 0 --steps $STEPS > gpurun_out/ab_A_$i.json 2>>gpurun_out/ab.err
cp $LIBB $L; python bench.py --config $CFG --no-cpu --no-check --no-compare --sustain-s 0 --steps $STEPS > gpurun_out/ab_B_$i.json 2>>gpurun_out/ab.err
done
cp /tmp/libA.so $L
tail -2 gpurun_out/ab.err
