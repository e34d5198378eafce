# Diagonal wide SYRK tiles without their empty column half: GPU suite, then same-box A/B against
# abtmp/libB.so at c3 / c4 (power_probe, under the cap) and c2 (bench line)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_gpu_fullsize_exact.py tests/test_gpu_leaf_schedule.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
L=paper_2101_01025_b200/libadjprod.so; cp $L /tmp/libA.so
: > gpurun_out/skip1.jsonl
for cfg in c3 c4; do for i in 1 2; do
  cp /tmp/libA.so $L; timeout 300 python tools/power_probe.py --config $cfg --seconds 5 --tag skip1 >> gpurun_out/skip1.jsonl 2>>gpurun_out/skip1.err
  cp abtmp/libB.so $L; timeout 300 python tools/power_probe.py --config $cfg --seconds 5 --tag full >> gpurun_out/skip1.jsonl 2>>gpurun_out/skip1.err
done; done
cp /tmp/libA.so $L
CFGS="c2" LIBB=abtmp/libB.so STEPS=20 bash tools/ab_multi.sh
