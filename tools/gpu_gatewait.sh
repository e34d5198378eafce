# Bounded claim-wave gate wait: full-size c3 / c4 parity and the scheduling variants, then same-box
# A/B against abtmp/libB.so at c3 / c4 under the power cap
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_gpu_fullsize_exact.py tests/test_gpu_leaf_schedule.py -x -q -m gpu > gpurun_out/gatewait_pytest.log 2>&1; echo pytest=$?
L=paper_2101_01025_b200/libadjprod.so; cp $L /tmp/libA.so
: > gpurun_out/gatewait.jsonl
for cfg in c3 c4; do for i in 1 2; do
  cp /tmp/libA.so $L; timeout 300 python tools/power_probe.py --config $cfg --seconds 5 --tag bounded >> gpurun_out/gatewait.jsonl 2>>gpurun_out/gatewait.err
  cp abtmp/libB.so $L; timeout 300 python tools/power_probe.py --config $cfg --seconds 5 --tag plain >> gpurun_out/gatewait.jsonl 2>>gpurun_out/gatewait.err
done; done
cp /tmp/libA.so $L
