#!/bin/bash
# Summarise one ncu report: key metrics + per-source-line stall/instruction mix.
# usage: tools/ncu_quick.sh report.ncu-rep [nlines]
R=$1; N=${2:-30}
ncu -i "$R" --page details --csv 2>/dev/null | python -c "
import csv,sys
keep=('Duration','Achieved Occupancy','Theoretical Occupancy','Registers Per Thread','Memory Throughput','DRAM Throughput','Compute (SM) Throughput','Issue Slots Busy','L1/TEX Hit Rate','L2 Hit Rate','Warp Cycles Per Issued Instruction','Executed Ipc Active','Block Limit Shared Mem','Block Limit Registers','Dynamic Shared Memory Per Block')
for r in csv.reader(sys.stdin):
    if len(r)>14 and r[12] in keep: print(r[12],r[14],r[13])
"
ncu -i "$R" --page source --print-source=cuda,sass --csv 2>/dev/null > /tmp/ncu_src.csv
python "$(dirname "$0")/ncu_lines.py" /tmp/ncu_src.csv "$N"
