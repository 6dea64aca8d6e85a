#!/bin/bash
# Hang/stability sweep: every IC schedule and the LT modes on the BASELINE graphs,
# each run under its own timeout (rc 124 = hang).
PASSES=${PASSES:-3}
for i in $(seq 1 $PASSES); do
  for spec in "cfg1 1048576 1" "cfg1 1048576 2" "cfg1 200000 3" "cfg3 1048576 1" "cfg3 262144 2" \
              "cfg3 262144 3" "cfg5 8192 2" "cfg5 8192 3" "cfg5 8192 1"; do
    set -- $spec
    timeout 60 python tools/profile_sampler.py $1 --sets $2 --ic-mode $3 > gpurun_out/s.log 2>&1
    echo "$i $1 n=$2 mode=$3 rc=$? $(tail -1 gpurun_out/s.log | grep -o "sample [0-9.]* ms")"
  done
  for spec in "cfg3c 2048 0" "cfg3c 512 3" "cfg5 8192 0"; do  # giant block schedule, dense rows
    set -- $spec
    timeout 120 python tools/profile_sampler.py $1 --sets $2 --ic-mode $3 > gpurun_out/s.log 2>&1
    echo "$i $1 n=$2 mode=$3 rc=$? $(tail -1 gpurun_out/s.log | grep -o "sample [0-9.]* ms")"
  done
  for c in cfg1 cfg2 cfg3 cfg4; do  # IMM: top-ups, cluster / grid selection
    timeout 120 python tools/profile_imm.py $c --repeat 2 > gpurun_out/s.log 2>&1
    echo "$i imm $c rc=$? $(tail -1 gpurun_out/s.log | grep -o "imm [0-9.]* ms")"
  done
  timeout 120 python tools/profile_sampler.py cfg5 --sets 32768 --ic-rng 1 > gpurun_out/s.log 2>&1
  echo "$i cfg5 fast rc=$? $(tail -1 gpurun_out/s.log | grep -o "sample [0-9.]* ms")"
  for spec in "cfg2 1048576 2" "cfg4 1048576 2" "cfg4 65536 1" "cfg4 65536 0"; do
    set -- $spec
    timeout 60 python tools/profile_sampler.py $1 --sets $2 --lt-scan $3 > gpurun_out/s.log 2>&1
    echo "$i $1 n=$2 scan=$3 rc=$? $(tail -1 gpurun_out/s.log | grep -o "sample [0-9.]* ms")"
  done
done
