#!/bin/bash
# dev sweep: bench lines for several configs / depths (no cpu leg, no parity check)
summ='import json,sys
for l in sys.stdin:
    l=l.strip()
    if not l.startswith("{"): continue
    d=json.loads(l); r=d["roofline"]
    print(d["config"]["workload"][:3], "d=%d" % d["config"]["depth"], "ms %.3f" % d["ms_per_step"], "val %.3e" % d["value"], "leaf %.3f" % r["frac"], "share", d["kernel_time_share"], "clk", d["clocks"]["sm_mhz"], d["clocks"]["reasons"], "W", d["clocks"].get("power_w_max"))'
for spec in "$@"; do
  cfg=${spec%:*}; dep=${spec#*:}
  timeout -s KILL 300 python bench.py --no-cpu --no-check --no-compare --config $cfg --depth $dep ${BENCH_EXTRA} --steps ${STEPS:-10} 2>/dev/null | python -c "$summ"
done
