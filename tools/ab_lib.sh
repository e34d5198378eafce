# Dev tool: A/B of the in-tree library against $LIBB (another build) on bench config $CFG, alternating
CFG=${CFG:-c2}; STEPS=${STEPS:-20}
for i in 1 2 3; do
python bench.py --config $CFG --no-cpu --no-check --no-compare --sustain-s 0 --steps $STEPS > gpurun_out/ab_A_$i.json 2>>gpurun_out/ab.err
ADJ_LIB_PATH=$LIBB python bench.py --config $CFG --no-cpu --no-check --no-compare --sustain-s 0 --steps $STEPS > gpurun_out/ab_B_$i.json 2>>gpurun_out/ab.err
done
tail -2 gpurun_out/ab.err
