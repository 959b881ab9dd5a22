bash tools/gpu_iter.sh k3b "rhs_parity or entropy_production or rk4 or full_size or eq56 or dense or dp54_step" C5
timeout 300 python tools/profile_run.py 3 12 8 2 > gpurun_out/k3b_prof_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"wadj3|rhs2_kernel" -s 2 -c 2 \
  -o gpurun_out/k3b_prof python tools/profile_run.py 3 12 8 2 > gpurun_out/k3b_ncu_full.log 2>&1; echo "ncu rc=$?"
