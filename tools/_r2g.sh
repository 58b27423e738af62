set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/r2g_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2g_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2g_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2g_smoke.log
timeout 900 python bench.py > gpurun_out/r2g_bench.jsonl 2> gpurun_out/r2g_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/r2g_bench_ref.jsonl 2> gpurun_out/r2g_bench_ref.err; echo "ref rc=$?"
for c in 5:k_el3d_fused 2:k_ac2d_fused 3:k_ac3d_fused 3f32:k_ac3d_fused32 4:k_el2d_fused; do
  cfg=${c%%:*}; k=${c##*:}; key=config$cfg; [ $cfg = 3f32 ] && key=config3_fp32
  timeout 600 ncu --replay-mode application --cache-control none --clock-control none \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:"$k<" -s 5 -c 12 --csv \
    --log-file gpurun_out/tw_$key.csv python tools/profile_config.py $cfg 20 > gpurun_out/tw_$key.log 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2g_launches.csv \
   python bench.py --steps 2 --warmup 1 --no-configs --no-cpu-baseline --nt 20 > gpurun_out/r2g_ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_el3d_fused -s 2 -c 1 \
   -o gpurun_out/r2g_el3f python tools/profile_config.py 5 4 > gpurun_out/r2g_ncu.log 2>&1
tail -3 gpurun_out/r2g_pytest.log; tail -2 gpurun_out/r2g_smoke.log; cut -c1-400 gpurun_out/r2g_bench.jsonl; tail -3 gpurun_out/r2g_bench.err
