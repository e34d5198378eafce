# Short launches: the default (wide, dynamic, gated) against the 256 x 256 leaf claimed dynamically
# with the gate (ADJ_LEAF_WIDE=0 ADJ_LEAF_DYNAMIC=1), c2 / c5 / x131071 bench lines, alternating
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in c2 c5 x131071; do for i in 1 2; do
  timeout 300 python bench.py --config $c --no-cpu --no-check --no-compare --sustain-s 0 --steps 20 > gpurun_out/nd_${c}_wide_$i.json 2>>gpurun_out/nd.err
  ADJ_LEAF_WIDE=0 ADJ_LEAF_DYNAMIC=1 timeout 300 python bench.py --config $c --no-cpu --no-check --no-compare --sustain-s 0 --steps 20 > gpurun_out/nd_${c}_narrowdyn_$i.json 2>>gpurun_out/nd.err
done; done
