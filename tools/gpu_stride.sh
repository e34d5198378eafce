# leaf DRAM traffic vs the arena's row stride: c3 shape (k = 32768, power-of-two strides) against
# k = 33792 (strides 132 / 66 x 128 B), same m, depth 2
for k in 32768 33792 34816; do
timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:leaf2_kernel -c 1 --csv python tools/run_one.py --config c3 --k $k --depth 2 --reps 1 --io16 > gpurun_out/ncu_stride_$k.csv 2>&1
grep -E "dram__bytes|hit_rate|duration" gpurun_out/ncu_stride_$k.csv | awk -F'","' -v t="k=$k" '{print t, $(NF-2), $(NF-1), $NF}'
done
