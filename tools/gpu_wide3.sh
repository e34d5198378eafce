# wide-N leaf: rasterisation band height (ADJ_BAND) 8 / 12 / 16
O=gpurun_out/wide3.log; : > $O
for c in c3 c4; do for b in 8 12 16 8 12 16; do
ADJ_LEAF_WIDE=1 ADJ_BAND=$b timeout 300 python tools/power_probe.py --config $c --tag ${c}_band$b >> $O 2>&1; done; done
grep '^{' $O | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['tag'], d['ms_per_call'], d['classes_ms']['leaf'], d['sm_mhz_median'], d['power_w_median'])"
for b in 8 12; do
ADJ_LEAF_WIDE=1 ADJ_BAND=$b timeout 600 ncu --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:leafw_kernel -c 1 --csv python tools/run_one.py --config c3 --reps 1 --io16 > gpurun_out/ncu_wband$b.csv 2>&1
grep -E "dram__bytes|hit_rate" gpurun_out/ncu_wband$b.csv | awk -F'","' -v t="band$b c3" '{print t, $(NF-2), $(NF-1), $NF}'
done
