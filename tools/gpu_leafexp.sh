python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for dbg in 0 3; do for shp in "8192 8192 8192" "18944 18944 2048" "18944 18944 8192" "9472 9472 16384"; do set -- $shp
ADJ_LEAF_DEBUG=$dbg timeout 120 python tools/time_leaf.py --m $1 --n $2 --k $3 2>&1 | tail -1
done; done > gpurun_out/leafexp.log 2>&1
