# wide-N leaf: 16 vs 8 epilogue warps vs the 256 x 256 leaf (back to back, alternating)
ADJ_LEAF_WIDE=2 timeout 120 python tools/wide_quick.py 2>&1 | tail -6
ADJ_LEAF_WIDE=2 ADJ_LEAFW_EPI=8 timeout 120 python tools/wide_quick.py 2>&1 | tail -2
O=gpurun_out/wide2.log; : > $O
for c in c3 c4; do for v in w16 w8 off w16 w8 off; do
case $v in w16) e="ADJ_LEAF_WIDE=1 ADJ_LEAFW_EPI=16";; w8) e="ADJ_LEAF_WIDE=1 ADJ_LEAFW_EPI=8";; off) e="ADJ_LEAF_WIDE=0";; esac
env $e timeout 300 python tools/power_probe.py --config $c --tag ${c}_$v >> $O 2>&1; done; done
grep '^{' $O | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['tag'], d['ms_per_call'], d['classes_ms']['leaf'], d['sm_mhz_median'], d['power_w_median'])"
