# Jacobian DMMA vs DFMA (same m8n8k4 formulation) A/B at configs[4], plus ncu of each
timeout 600 python scripts/jac_ab.py
LT_LIB=paper_1409_2556_b200/_lib/liblaptomo_gpu_dfma.so timeout 900 python scripts/jac_ab.py
timeout 900 ncu --set full --clock-control none -k regex:jacobian_mma4 -c 1 -o gpurun_out/r2_jac_dmma -f python scripts/jac_ab.py > gpurun_out/r2_jac_dmma.log 2>&1
LT_LIB=paper_1409_2556_b200/_lib/liblaptomo_gpu_dfma.so timeout 1200 ncu --set full --clock-control none -k regex:jacobian_mma4 -c 1 -o gpurun_out/r2_jac_dfma -f python scripts/jac_ab.py > gpurun_out/r2_jac_dfma.log 2>&1
ls -la gpurun_out/r2_jac_*
