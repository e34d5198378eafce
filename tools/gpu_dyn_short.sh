# Dynamic claiming (and so the claim-wave gate) forced on the short launches (ADJ_LEAF_DYNAMIC=1)
# against their static default: c2 / c5 / x131071 / q5 bench lines, alternating on one box
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in c2 c5 x131071; do for i in 1 2; do
  timeout 300 python bench.py --config $c --no-cpu --no-check --no-compare --sustain-s 0 --steps 20 > gpurun_out/ds_${c}_static_$i.json 2>>gpurun_out/ds.err
  ADJ_LEAF_DYNAMIC=1 timeout 300 python bench.py --config $c --no-cpu --no-check --no-compare --sustain-s 0 --steps 20 > gpurun_out/ds_${c}_dyn_$i.json 2>>gpurun_out/ds.err
done; done
