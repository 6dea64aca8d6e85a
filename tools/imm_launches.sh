#!/bin/bash
# IMM table on all configs + ncu launch lists of run_imm (cfg1, cfg3, cfg4).
mkdir -p gpurun_out
timeout 900 python tools/imm_table.py > gpurun_out/imm_table.jsonl 2> gpurun_out/imm_table.err; echo imm_table rc=$?
for c in cfg4 cfg1 cfg3; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/imm_launches_$c.csv python tools/profile_imm.py $c --repeat 1 > gpurun_out/imm_launches_$c.log 2>&1
  echo $c rc=$?
done
