for k in 1 2 3; do timeout 300 python tools/pipe_probe.py matmul 131072 24 32 2>&1 | head -6; done
timeout 300 python bench.py --no-cpu | cut -c1-300
