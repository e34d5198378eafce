# Dev tool: A/B of the in-tree library against $LIBB over several bench configs ($CFGS), alternating
for c in ${CFGS:-c2 c5 q5 x65521}; do
for i in 1 2; do
python bench.py --config $c --no-cpu --no-check --no-compare --sustain-s 0 --steps ${STEPS:-10} > gpurun_out/ab_${c}_A_$i.json 2>>gpurun_out/ab.err
ADJ_LIB_PATH=$LIBB python bench.py --config $c --no-cpu --no-check --no-compare --sustain-s 0 --steps ${STEPS:-10} > gpurun_out/ab_${c}_B_$i.json 2>>gpurun_out/ab.err
done; done
tail -2 gpurun_out/ab.err
