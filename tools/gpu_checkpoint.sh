#!/bin/bash
# GPU checkpoint (run under gpurun): full GPU suite, both bench arms, then the ncu launch
# list and one --set full capture of the headline (config-5) step kernel, each ncu pass only
# after its own command exited 0 without ncu.  Outputs in gpurun_out/; summarise locally with
# python tools/summarize_profiles.py <tag>.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/ck_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ck_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ck_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/ck_smoke.log
timeout 900 python bench.py > gpurun_out/ck_bench.jsonl 2> gpurun_out/ck_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/ck_bench_ref.jsonl 2> gpurun_out/ck_bench_ref.err; echo "ref rc=$?"
if python tools/profile_config.py 5 14 > gpurun_out/ck_step.log 2>&1; then
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/ck_launches_raw.csv python tools/profile_config.py 5 14 > /dev/null 2>&1
  ncu --set full --clock-control none --import-source on -k regex:k_el3d_fused -s 5 -c 1 \
      -o gpurun_out/ck_el3d_full python tools/profile_config.py 5 14 > gpurun_out/ck_ncu.log 2>&1
fi
tail -3 gpurun_out/ck_pytest.log; tail -2 gpurun_out/ck_smoke.log; cat gpurun_out/ck_bench.jsonl | cut -c1-300
