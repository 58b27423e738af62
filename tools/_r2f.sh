set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_elastic3d_fused.py -x -q > gpurun_out/r2f_el3f.log 2>&1; echo "el3f rc=$?" >> gpurun_out/r2f_el3f.log
timeout 300 python tools/measure_configs.py 50 5 --opt fused_el3=1 | cut -c1-200 > gpurun_out/r2f_c5.jsonl 2>&1
python - >> gpurun_out/r2f_c5.jsonl 2>&1 <<'PY'
import sys; sys.path.insert(0, "."); sys.argv = ["x"]
import tools.measure_configs as mc, paper_2310_00236_b200 as hw
s = mc.cfg5(); s.upload(s.new_state())
lib = hw._abi.load()
print("div modes rho_x rho_s rho_m:", [lib.hw_plane_div_mode(s._lib_handle(), p) for p in (0, 1, 2)])
PY
tail -2 gpurun_out/r2f_el3f.log; cat gpurun_out/r2f_c5.jsonl
