# pure tcgen05 kind::i8 rate (operands resident in smem, random bytes) back to back for 10 s with
# NVML clocks / power sampled, then the c3 leaf under the same cap (tools/power_probe.py)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/mma_peak_bin tools/mma_peak.cu || exit 1
nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.active --format=csv,noheader -lms 100 > gpurun_out/smi_mma.csv &
SMI=$!
/tmp/mma_peak_bin sustain 20000 10 > gpurun_out/mma_sustain.json
kill $SMI
/tmp/mma_peak_bin 20000 > gpurun_out/mma_burst.json
python tools/power_probe.py --config c3 --seconds 6 --tag c3 > gpurun_out/c3_probe.json 2>&1
cat gpurun_out/mma_sustain.json gpurun_out/mma_burst.json; grep '^{' gpurun_out/c3_probe.json
python - <<'PY'
import statistics
rows=[l.split(',') for l in open('gpurun_out/smi_mma.csv') if l.strip()]
clk=[float(r[0].split()[0]) for r in rows]; pw=[float(r[1].split()[0]) for r in rows]
n=len(rows); tail=slice(n//2, n)
print({"samples": n, "sm_mhz_median_2nd_half": statistics.median(clk[tail]), "power_w_median_2nd_half": statistics.median(pw[tail]), "reasons": sorted(set(r[2].strip() for r in rows[n//2:]))})
PY
