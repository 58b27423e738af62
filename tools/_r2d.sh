set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_elastic3d_fused.py -x -q > gpurun_out/r2d_el3f.log 2>&1; echo "el3f rc=$?" >> gpurun_out/r2d_el3f.log
for g in 1 2 4; do timeout 300 python tools/measure_configs.py 50 5 --opt fused_el3=1 --opt el3_group=$g | cut -c1-200; done > gpurun_out/r2d_c5.jsonl 2>&1
timeout 300 python tools/measure_configs.py 50 5 --lib paper_2310_00236_b200/lib/variants/lib_c8.so --opt fused_el3=1 | cut -c1-200 >> gpurun_out/r2d_c5.jsonl 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_el3d_fused -s 2 -c 1 \
   -o gpurun_out/r2d_f4 python tools/profile_config.py --opt fused_el3=1 5 4 > gpurun_out/r2d_ncu.log 2>&1
tail -2 gpurun_out/r2d_el3f.log; cat gpurun_out/r2d_c5.jsonl
