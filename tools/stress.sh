#!/bin/bash
# Hang/stability sweep: every IC schedule and the LT modes on the BASELINE graphs,
# each run under its own timeout (rc 124 = hang).
for i in 1 2 3; do
  for spec in "cfg1 1048576 1" "cfg1 1048576 2" "cfg1 200000 3" "cfg3 1048576 1" "cfg3 262144 2" \
              "cfg3 262144 3" "cfg5 8192 2" "cfg5 8192 3" "cfg5 8192 1"; do
    set -- $spec
    timeout 60 python tools/profile_sampler.py $1 --sets $2 --ic-mode $3 > gpurun_out/s.log 2>&1
    echo "$i $1 n=$2 mode=$3 rc=$? $(tail -1 gpurun_out/s.log | grep -o "sample [0-9.]* ms")"
  done
  for spec in "cfg2 1048576 2" "cfg4 1048576 2" "cfg4 65536 1" "cfg4 65536 0"; do
    set -- $spec
    timeout 60 python tools/profile_sampler.py $1 --sets $2 --lt-scan $3 > gpurun_out/s.log 2>&1
    echo "$i $1 n=$2 scan=$3 rc=$? $(tail -1 gpurun_out/s.log | grep -o "sample [0-9.]* ms")"
  done
done
