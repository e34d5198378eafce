# K1 A/B: the in-tree library (A) against abtmp/libB.so (B) under the power cap at c3 / c4
# (power_probe.py, alternating), after the fused-K1 parity tests; then the PCIe probe.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_k1_fused.py -x -q -m gpu > gpurun_out/k1ab_pytest.log 2>&1; echo pytest=$?
L=paper_2101_01025_b200/libadjprod.so; cp $L /tmp/libA.so
: > gpurun_out/k1ab.jsonl
for cfg in ${CFGS:-c3 c4}; do for i in 1 2; do
  cp /tmp/libA.so $L; timeout 300 python tools/power_probe.py --config $cfg --seconds 5 --tag A >> gpurun_out/k1ab.jsonl 2>>gpurun_out/k1ab.err
  cp abtmp/libB.so $L; timeout 300 python tools/power_probe.py --config $cfg --seconds 5 --tag B >> gpurun_out/k1ab.jsonl 2>>gpurun_out/k1ab.err
done; done
cp /tmp/libA.so $L
timeout 300 python tools/pcie_probe.py --compute > gpurun_out/pcie.jsonl 2>gpurun_out/pcie.err; echo pcie=$?
