export SFG_TAIL_MINB=16 CAPS=32768 DEPTHS= STEPS=1
timeout 300 ncu --set full --clock-control none -k regex:sfg_jit -s 4 -c 2 -o gpurun_out/ab_old python abtest/old/tools/exec_probe.py matmul 65536 > gpurun_out/ab_ncu_old.log 2>&1
SFG_GROUP=1 timeout 300 ncu --set full --clock-control none -k regex:sfg_jit -s 6 -c 3 -o gpurun_out/ab_new python tools/exec_probe.py matmul 65536 > gpurun_out/ab_ncu_new.log 2>&1
