# L2 cache policies on the leaf's TMA loads (ADJ_LEAF_DEBUG 1024: A evict_last, 2048: B evict_first)
O=gpurun_out/hint.log; : > $O
for c in c3 c4; do for d in 0 1024 3072 2048 0 1024 3072; do
ADJ_LEAF_DEBUG=$d python tools/power_probe.py --config $c --tag ${c}_hint$d >> $O 2>&1; done; done
grep '^{' $O | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['tag'], d['ms_per_call'], d['classes_ms']['leaf'], d['sm_mhz_median'], d['power_w_median'])"
for d in 0 1024 3072; do
ADJ_LEAF_DEBUG=$d timeout 600 ncu --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:leaf2_kernel -c 1 --csv python tools/run_one.py --config c3 --reps 1 --io16 > gpurun_out/ncu_hint$d.csv 2>&1
grep -E "dram__bytes|hit_rate" gpurun_out/ncu_hint$d.csv | awk -F'","' -v t="hint$d c3" '{print t, $(NF-2), $(NF-1), $NF}'
done
