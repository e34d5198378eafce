# Dev tool: A/B of the in-tree library against $LIBB over several bench configs ($CFGS), alternating
# (the product binding loads only the in-tree libadjprod.so, so the two builds are swapped into place)
L=paper_2101_01025_b200/libadjprod.so; cp $L /tmp/libA.so
for c in ${CFGS:-c2 c5 q5 x65521}; do
for i in 1 2; do
cp /tmp/libA.so $L; python bench.py --config $c --no-cpu --no-check --no-compare --sustain-s 0 --steps ${STEPS:-10} > gpurun_out/ab_${c}_A_$i.json 2>>gpurun_out/ab.err
cp $LIBB $L; python bench.py --config $c --no-cpu --no-check --no-compare --sustain-s 0 --steps ${STEPS:-10} > gpurun_out/ab_${c}_B_$i.json 2>>gpurun_out/ab.err
done; done
cp /tmp/libA.so $L
tail -2 gpurun_out/ab.err
