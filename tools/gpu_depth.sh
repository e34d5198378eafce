# depth re-check under the power cap (fused K1 in place): c3 / c4 at depths 1, 2, 3, back to back
O=gpurun_out/depth.log; : > $O
for d in 2 1 3 2; do python tools/power_probe.py --config c3 --depth $d --tag c3d$d >> $O 2>&1; done
for d in 2 1 3 2; do python tools/power_probe.py --config c4 --depth $d --tag c4d$d >> $O 2>&1; done
