# low-memory schedule: GPU tests, then same-box A/B against the grouped schedule at c3 / c4
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_lowmem.py -x -q > gpurun_out/pytest_lowmem.log 2>&1; echo pytest=$?
O=gpurun_out/lowmem.log; : > $O
for i in 1 2; do
python tools/power_probe.py --config c3 --tag grouped >> $O 2>&1
python tools/power_probe.py --config c3 --lowmem --tag lowmem >> $O 2>&1
python tools/power_probe.py --config c4 --tag grouped >> $O 2>&1
python tools/power_probe.py --config c4 --lowmem --tag lowmem >> $O 2>&1
done
python tools/power_probe.py --config c2 --depth 1 --tag grouped_c2d1 >> $O 2>&1
python tools/power_probe.py --config c2 --depth 1 --lowmem --tag lowmem_c2d1 >> $O 2>&1
