export CUDA_DEVICE_MAX_CONNECTIONS=32
for mb in 12 16; do for d in 16 32; do
echo "== minb=$mb d=$d"; SFG_TAIL_MINB=$mb timeout 300 python tools/pipe_probe.py matmul 65536 $d 96 2>&1| head -3
done; done
