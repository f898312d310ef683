#!/bin/bash
# Runs on the GPU box (gpurun): bench lines, ncu launch list of the bench
# command, and one `ncu --set full` capture of each config's dominant kernel.
set -u
OUT=gpurun_out/prof
mkdir -p $OUT
timeout 300 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
for c in 1 3 4 5; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_cfg$c.json 2> $OUT/bench_cfg$c.err
done
# launch list of the default bench command (short run; numbers under ncu are not bench values)
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/plain.log 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_bench_cfg2.csv \
    timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/ncu_launches.log 2>&1
# full captures of the dominant kernels
cap() {  # name config scale regex skip
  timeout 300 python tools/profile_step.py --config $2 --scale $3 --steps 2 > $OUT/plain_$1.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$4" -s $5 -c 1 -o $OUT/$1 \
      timeout 300 python tools/profile_step.py --config $2 --scale $3 --steps 2 > $OUT/ncu_$1.log 2>&1
}
cap spadd_tiles 2 1.0 spadd_tiles 1
cap spgemm_cfg1_hashM1 1 1.0 hash_numeric 1
cap spgemm_cfg3_long 3 1.0 long_numeric 0
cap spgemm_cfg3_hashM 3 1.0 hash_numeric 3
cap mttkrp_dense32 4 1.0 mttkrp_dense32q 0
cap mttkrp_sparse 5 1.0 mttkrp_sparse 0
ls -la $OUT
