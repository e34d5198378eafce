# K4 A/B (in-tree library vs abtmp/libB.so) at c3 / c4 under the power cap, after the full GPU suite
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
L=paper_2101_01025_b200/libadjprod.so; cp $L /tmp/libA.so
: > gpurun_out/k4ab.jsonl
for cfg in ${CFGS:-c3 c4}; do for i in 1 2; do
  cp /tmp/libA.so $L; timeout 300 python tools/power_probe.py --config $cfg --seconds 5 --tag A >> gpurun_out/k4ab.jsonl 2>>gpurun_out/k4ab.err
  cp abtmp/libB.so $L; timeout 300 python tools/power_probe.py --config $cfg --seconds 5 --tag B >> gpurun_out/k4ab.jsonl 2>>gpurun_out/k4ab.err
done; done
cp /tmp/libA.so $L
