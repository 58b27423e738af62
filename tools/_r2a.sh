set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_elastic3d_fused.py -x -q > gpurun_out/r2a_el3f.log 2>&1; echo "el3f rc=$?" >> gpurun_out/r2a_el3f.log
timeout 300 python tools/measure_configs.py 50 5 --opt fused_el3=1 > gpurun_out/r2a_c5f.jsonl 2>&1
timeout 300 python tools/measure_configs.py 50 5 > gpurun_out/r2a_c5s.jsonl 2>&1
timeout 1200 python -m pytest tests/test_gpu_production.py -x -q -rA > gpurun_out/r2a_prod.log 2>&1; echo "prod rc=$?" >> gpurun_out/r2a_prod.log
tail -3 gpurun_out/r2a_el3f.log; cat gpurun_out/r2a_c5f.jsonl gpurun_out/r2a_c5s.jsonl | cut -c1-250; tail -5 gpurun_out/r2a_prod.log
