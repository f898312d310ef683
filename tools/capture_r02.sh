#!/bin/bash
# Round-2 evidence, run on the GPU box (gpurun): full GPU suite, bench lines (all
# five configs, reference arm, NCCL world-1), the ncu launch list of the bench
# command and `ncu --set full` captures of config 5's kernels.
set -u
OUT=gpurun_out/r02
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -5 > $OUT/gputest.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1 > $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench_all.json 2> $OUT/bench_all.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_reference_cfg5.json 2> $OUT/bench_reference.err
for c in 3 5; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 2951$c \
      bench.py --gpus 1 --config $c --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_torchrun1_cfg$c.json 2> $OUT/bench_torchrun1_cfg$c.err
done
# launch lists of the bench command, one per config (short runs; numbers under ncu are not bench values)
for c in 1 2 3 4 5; do
  timeout 300 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > $OUT/plain_cfg$c.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $OUT/launches_bench_cfg$c.csv \
      python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > $OUT/ncu_l$c.log 2>&1
done
cap() {  # name config regex skip
  timeout 300 python tools/profile_step.py --config $2 --steps 2 > $OUT/plain_$1.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$3" -s $4 -c 1 -o $OUT/$1 \
      python tools/profile_step.py --config $2 --steps 2 > $OUT/ncu_$1.log 2>&1
}
cap mttkrp_sparse_filter 5 mttkrp_sparse_filter 1
cap mttkrp_sparse_expand 5 mttkrp_sparse_expand 1
cap mttkrp_sparse_accum 5 mttkrp_sparse_accum 1
cap spgemm_bucketM 3 bucket_numeric 3
cap spgemm_long 3 long_numeric 0
ls -la $OUT
