# Lazy intermediate Horner steps of the wide leaf: parity (full-size c3 / c4, scheduling variants,
# fused-K1 suite), then same-box A/B against abtmp/libB.so at c3 / c4 under the power cap
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_fullsize_exact.py tests/test_gpu_leaf_schedule.py tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/lazy_pytest.log 2>&1; echo pytest=$?
L=paper_2101_01025_b200/libadjprod.so; cp $L /tmp/libA.so
: > gpurun_out/lazy.jsonl
for cfg in c3 c4; do for i in 1 2; do
  cp /tmp/libA.so $L; timeout 300 python tools/power_probe.py --config $cfg --seconds 5 --tag lazy >> gpurun_out/lazy.jsonl 2>>gpurun_out/lazy.err
  cp abtmp/libB.so $L; timeout 300 python tools/power_probe.py --config $cfg --seconds 5 --tag full >> gpurun_out/lazy.jsonl 2>>gpurun_out/lazy.err
done; done
cp /tmp/libA.so $L
