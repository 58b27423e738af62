set -u
mkdir -p gpurun_out
V=paper_2310_00236_b200/lib/variants/lib_c4.so
timeout 300 python tools/measure_configs.py 50 5 --opt fused_el3=1 --lib $V > gpurun_out/r2b_c5f4.jsonl 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_el3d_fused -s 2 -c 1 \
   -o gpurun_out/r2b_f8 python tools/profile_config.py --opt fused_el3=1 5 4 > gpurun_out/r2b_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_el3d_fused -s 2 -c 1 \
   -o gpurun_out/r2b_f4 python tools/profile_config.py --lib $V --opt fused_el3=1 5 4 >> gpurun_out/r2b_ncu.log 2>&1
cat gpurun_out/r2b_c5f4.jsonl | cut -c1-200
