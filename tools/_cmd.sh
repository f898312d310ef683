mkdir -p gpurun_out/ll
python -m pytest tests/test_gpu_spgemm.py tests/test_gpu_golden.py tests/test_gpu_modes.py -x -q 2>&1 | tail -3
python bench.py --config 3 --no-cpu-baseline --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); print(d['ms_per_step'], d['kernels_total_ms'], d['roofline']['frac'])"
python tools/profile_step.py --config 3 --steps 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ll/launch_cfg3.csv python tools/profile_step.py --config 3 --steps 1 > /dev/null 2>&1
