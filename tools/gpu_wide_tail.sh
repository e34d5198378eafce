# wide-N tail K-split (ADJ_WIDE_TAIL): parity with it on (full GPU suite; every launch wide), then
# a same-box A/B of the short-launch configs and c3
O=gpurun_out/wtail; mkdir -p $O
ADJ_WIDE_TAIL=1 timeout 1200 python -m pytest tests -m gpu -x -q > $O/suite_tail1.log 2>&1; echo suite_tail1=$?; tail -2 $O/suite_tail1.log
ADJ_LEAF_WIDE=2 ADJ_WIDE_TAIL=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -x -q > $O/parity_w2_tail1.log 2>&1; echo parity_w2_tail1=$?; tail -2 $O/parity_w2_tail1.log
ADJ_LEAF_WIDE=2 ADJ_WIDE_TAIL=0 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -x -q > $O/parity_w2_tail0.log 2>&1; echo parity_w2_tail0=$?; tail -2 $O/parity_w2_tail0.log
for r in 1 2; do
  for c in c2 c5 q5 x131071 c3; do
    for t in 0 1; do
      ADJ_WIDE_TAIL=$t timeout 300 python bench.py --config $c --steps 20 --no-cpu --no-check --no-compare --sustain-s 0 > $O/ab_${c}_t${t}_r$r.log 2>&1
    done
  done
done
python - <<'P'
import json,glob,re
rows={}
for f in sorted(glob.glob('gpurun_out/wtail/ab_*.log')):
    l=[x for x in open(f) if x.startswith('{')]
    m=re.search(r'ab_(\w+?)_t(\d)_r(\d)',f)
    if not l: print(f,'NO LINE'); continue
    d=json.loads(l[-1])
    print(m.group(1),'tail',m.group(2),'round',m.group(3),'ms',round(d['ms_per_step'],4),'leaf_ms',round(d['roofline']['leaf_ms_per_launch'],4),'launches',d['gpu_launches'],'clk',d['clocks']['sm_mhz'])
P
