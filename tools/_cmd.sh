python -m pytest tests/test_gpu_spadd.py tests/test_gpu_golden.py tests/test_gpu_modes.py -x -q 2>&1 | tail -3
python bench.py --no-cpu-baseline --steps 100 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); print(d['ms_per_step'], d['kernels_total_ms'], d['roofline']['frac'])"
mkdir -p gpurun_out/ll
python tools/profile_step.py --config 2 --steps 2 > gpurun_out/ll/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:spadd_tiles -s 1 -c 1 -o gpurun_out/ll/spadd_tiles2 python tools/profile_step.py --config 2 --steps 2 > gpurun_out/ll/ncu_spadd.log 2>&1
