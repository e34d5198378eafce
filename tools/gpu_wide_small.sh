# Wide-N leaf forced on the short launches (ADJ_LEAF_WIDE=2) against the default (256 x 256 below
# 16 waves): c2 / c5 / x131071 bench lines, alternating on one box
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in c2 c5 x131071; do for i in 1 2; do
  timeout 300 python bench.py --config $c --no-cpu --no-check --no-compare --sustain-s 0 --steps 20 > gpurun_out/ws_${c}_def_$i.json 2>>gpurun_out/ws.err
  ADJ_LEAF_WIDE=2 timeout 300 python bench.py --config $c --no-cpu --no-check --no-compare --sustain-s 0 --steps 20 > gpurun_out/ws_${c}_wide_$i.json 2>>gpurun_out/ws.err
done; done
