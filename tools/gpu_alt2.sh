# K-direction alternation + mixed-middle accumulator order as defaults: GPU suite, then same-box
# A/B against ADJ_LEAF_KALT=0 ADJ_ACC_ORDER=0 at c3 / c4 (power_probe) and c2 / q5 (bench lines)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
: > gpurun_out/alt2.jsonl
for cfg in c3 c4; do for rep in 1 2; do
  timeout 300 python tools/power_probe.py --config $cfg --seconds 5 --tag new >> gpurun_out/alt2.jsonl 2>>gpurun_out/alt2.err
  ADJ_LEAF_KALT=0 ADJ_ACC_ORDER=0 timeout 300 python tools/power_probe.py --config $cfg --seconds 5 --tag old >> gpurun_out/alt2.jsonl 2>>gpurun_out/alt2.err
done; done
for c in c2 q5; do for rep in 1 2; do
  timeout 300 python bench.py --config $c --no-cpu --no-check --no-compare --sustain-s 0 --steps 20 > gpurun_out/alt2_${c}_new_$rep.json 2>>gpurun_out/alt2.err
  ADJ_LEAF_KALT=0 ADJ_ACC_ORDER=0 timeout 300 python bench.py --config $c --no-cpu --no-check --no-compare --sustain-s 0 --steps 20 > gpurun_out/alt2_${c}_old_$rep.json 2>>gpurun_out/alt2.err
done; done
