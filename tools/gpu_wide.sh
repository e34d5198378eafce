# wide-N leaf (ADJ_LEAF_WIDE: 0 off, 1 long launches, 2 always): parity suite with it forced, A/B
ADJ_LEAF_WIDE=2 timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_wide.log 2>&1; echo pytest_wide=$?; tail -3 gpurun_out/pytest_wide.log
O=gpurun_out/wide.log; : > $O
for c in c3 c4; do for w in 1 0 1 0; do ADJ_LEAF_WIDE=$w timeout 300 python tools/power_probe.py --config $c --tag ${c}_wide$w >> $O 2>&1; done; done
for w in 2 0 2 0; do ADJ_LEAF_WIDE=$w timeout 300 python tools/power_probe.py --config c2 --seconds 3 --tag c2_wide$w >> $O 2>&1; done
grep '^{' $O | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['tag'], d['ms_per_call'], d['classes_ms']['leaf'], d['sm_mhz_median'], d['power_w_median'])"
