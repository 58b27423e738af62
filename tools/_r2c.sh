set -u
mkdir -p gpurun_out
V=paper_2310_00236_b200/lib/variants/lib_c4.so
python tools/profile_config.py --lib $V --opt fused_el3=1 5 4 > gpurun_out/r2c_plain.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_el3d_fused -s 2 -c 1 \
   -o gpurun_out/r2c_f4 python tools/profile_config.py --lib $V --opt fused_el3=1 5 4 >> gpurun_out/r2c_ncu.log 2>&1
cat gpurun_out/r2c_plain.log
