# Leaf rasterisation band height (ADJ_BAND, diagnostics) at c3 / c4 under the power cap:
# power_probe.py back to back, the values alternating with the default (8) as control.
# Output: gpurun_out/band.jsonl
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
: > gpurun_out/band.jsonl
for cfg in ${CFGS:-c3 c4}; do
  for rep in 1 2; do
    for b in ${BANDS:-8 4 12 16 24}; do
      ADJ_BAND=$b timeout 300 python tools/power_probe.py --config $cfg --seconds ${SECS:-5} --tag band$b >> gpurun_out/band.jsonl 2> gpurun_out/band_err.log
    done
  done
done
