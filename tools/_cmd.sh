mkdir -p gpurun_out/ll
timeout 200 python -m pytest tests/test_gpu_mttkrp.py tests/test_gpu_golden.py -x -q 2>&1 | tail -2
timeout 120 python bench.py --config 4 --no-cpu-baseline --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); print(d['ms_per_step'], d['kernels_total_ms'], d['roofline']['frac'])"
