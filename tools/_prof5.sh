set -u
mkdir -p gpurun_out
export HALFWAVE_FUSED_EL3=1
python tools/profile_config.py 5 4 > gpurun_out/p5_plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_el3d_fused -s 2 -c 1 \
   -o gpurun_out/p5_fused python tools/profile_config.py 5 4 > gpurun_out/p5_ncu.log 2>&1
unset HALFWAVE_FUSED_EL3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_el3d_ -s 2 -c 2 \
   -o gpurun_out/p5_stream python tools/profile_config.py 5 4 >> gpurun_out/p5_ncu.log 2>&1
echo rc=$?
