# e2e pipeline A/B on one box: two A buffers (previous bench) vs three A buffers + io-only bound
for r in 1 2; do
  timeout 600 python tools/bench_prev.py --no-cpu --no-check --no-compare --sustain-s 0 > gpurun_out/e2e_prev_$r.log 2>&1; echo prev=$?
  timeout 600 python bench.py --no-cpu --no-check --no-compare --sustain-s 0 > gpurun_out/e2e_new_$r.log 2>&1; echo new=$?
done
python - <<'P'
import json,glob
for f in sorted(glob.glob('gpurun_out/e2e_*.log')):
    l=[x for x in open(f) if x.startswith('{')]
    if not l: print(f,'no line'); continue
    d=json.loads(l[-1]); e=d['e2e']
    print(f, 'dev', round(d['ms_per_step'],2), 'e2e', round(e['ms_per_step'],2), 'io', e.get('io_only_ms'), 'frac', e.get('frac_of_bound'))
P
