# c4 depth 2 vs 3 alternating (3 each), x16k depth 1 vs 2
O=gpurun_out/depth2.log; : > $O
for d in 3 2 3 2 3 2; do python tools/power_probe.py --config c4 --depth $d --seconds 6 --tag c4d$d >> $O 2>&1; done
for d in 1 2 1 2; do python tools/power_probe.py --config x16k --depth $d --tag x16kd$d >> $O 2>&1; done
