# Fused K1 storing both K halves of a thread as one 8-byte word (permuted K columns): parity of the
# fused K1 / full-size / scheduling / parity suites, then same-box A/B against abtmp/libB.so
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_gpu_k1_fused.py tests/test_gpu_fullsize_exact.py tests/test_gpu_parity.py tests/test_gpu_lowmem.py -x -q -m gpu > gpurun_out/k1v2_pytest.log 2>&1; echo pytest=$?
L=paper_2101_01025_b200/libadjprod.so; cp $L /tmp/libA.so
: > gpurun_out/k1v2.jsonl
for cfg in c3 c4; do for i in 1 2; do
  cp /tmp/libA.so $L; timeout 300 python tools/power_probe.py --config $cfg --seconds 5 --tag v2 >> gpurun_out/k1v2.jsonl 2>>gpurun_out/k1v2.err
  cp abtmp/libB.so $L; timeout 300 python tools/power_probe.py --config $cfg --seconds 5 --tag v1 >> gpurun_out/k1v2.jsonl 2>>gpurun_out/k1v2.err
done; done
cp /tmp/libA.so $L
