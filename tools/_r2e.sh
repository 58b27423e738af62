set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_elastic3d_fused.py -x -q > gpurun_out/r2e_el3f.log 2>&1; echo "el3f rc=$?" >> gpurun_out/r2e_el3f.log
timeout 300 python tools/measure_configs.py 50 5 --opt fused_el3=1 | cut -c1-200 > gpurun_out/r2e_c5.jsonl 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_el3d_fused -s 2 -c 1 \
   -o gpurun_out/r2e_f4 python tools/profile_config.py --opt fused_el3=1 5 4 > gpurun_out/r2e_ncu.log 2>&1
tail -2 gpurun_out/r2e_el3f.log; cat gpurun_out/r2e_c5.jsonl
