# Wide launches always dynamic (gated): GPU suite, then same-box A/B against abtmp/libB.so on the
# short wide launches (c2, c5, x131071) and q5
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
CFGS="c2 c5 x131071 q5" LIBB=abtmp/libB.so STEPS=20 bash tools/ab_multi.sh
