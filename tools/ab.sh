export SFG_TAIL_MINB=16 CUDA_DEVICE_MAX_CONNECTIONS=32
for d in 16 24; do
echo "== G=1 d=$d"; SFG_GROUP=1 timeout 300 python tools/pipe_probe.py matmul 65536 $d 64 2>&1| head -3
echo "== tailG=8 d=$d"; SFG_GROUP=8 timeout 300 python tools/pipe_probe.py matmul 65536 $d 64 2>&1| head -3
done
echo "== bulkG=8 d=24"; SFG_BULK_GROUP=8 SFG_GROUP=8 timeout 300 python tools/pipe_probe.py matmul 65536 24 64 2>&1| head -3
