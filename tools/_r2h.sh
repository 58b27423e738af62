set -u
mkdir -p gpurun_out
for c in 5:k_el3d_fused 2:k_ac2d_fused 3:k_ac3d_fused 3f32:k_ac3d_fused32 4:k_el2d_fused; do
  cfg=${c%%:*}; k=${c##*:}; key=config$cfg; [ $cfg = 3f32 ] && key=config3_fp32
  timeout 600 ncu --replay-mode application --cache-control none --clock-control none \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k "regex:^${k}\$" -s 5 -c 12 --csv \
    --log-file gpurun_out/tw_$key.csv python tools/profile_config.py $cfg 20 > gpurun_out/tw_$key.log 2>&1
done
wc -l gpurun_out/tw_*.csv
