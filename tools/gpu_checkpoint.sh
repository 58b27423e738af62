#!/bin/bash
# GPU checkpoint (run under gpurun): full GPU suite, smoke, both bench arms, then -- each ncu pass only
# after its own command exited 0 without ncu -- the ncu launch list of a short bench run, one --set full
# capture of the headline (config-5) step kernel and the steady-state DRAM traffic windows of every
# config's step kernel.  Outputs in gpurun_out/; summarise locally with
#   python tools/launch_summary.py gpurun_out/ck_launches_raw.csv profiles/<tag>_launches.csv "<title>"
#   python tools/ncu_summary.py gpurun_out/ck_el3d_full.ncu-rep "<title>" 134217728
#   python tools/traffic_window.py <tag> gpurun_out/tw_config*.csv
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/ck_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ck_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ck_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/ck_smoke.log
timeout 900 python bench.py > gpurun_out/ck_bench.jsonl 2> gpurun_out/ck_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/ck_bench_ref.jsonl 2> gpurun_out/ck_bench_ref.err; echo "ref rc=$?"
SHORT="bench.py --steps 2 --warmup 1 --no-configs --no-cpu-baseline --nt 20"
if timeout 600 python $SHORT > gpurun_out/ck_short.jsonl 2>&1; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file gpurun_out/ck_launches_raw.csv python $SHORT > /dev/null 2>&1
fi
if python tools/profile_config.py 5 8 > gpurun_out/ck_step.log 2>&1; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_el3d_fused -s 4 -c 1 \
      -o gpurun_out/ck_el3d_full python tools/profile_config.py 5 8 > gpurun_out/ck_ncu.log 2>&1
fi
W="--replay-mode application --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -s 5 -c 12 --csv"
for pair in "2:k_ac2d_fused:config2" "3:k_ac3d_fused:config3" "3f32:k_ac3d_fused32:config3_fp32" "4:k_el2d_fused:config4" "5:k_el3d_fused:config5"; do
  IFS=: read c k name <<< "$pair"
  if python tools/profile_config.py $c 20 > /dev/null 2>&1; then
    timeout 900 ncu $W -k regex:$k --log-file gpurun_out/tw_$name.csv python tools/profile_config.py $c 20 > /dev/null 2>&1
  fi
done
tail -3 gpurun_out/ck_pytest.log; tail -2 gpurun_out/ck_smoke.log; cut -c1-300 gpurun_out/ck_bench.jsonl
