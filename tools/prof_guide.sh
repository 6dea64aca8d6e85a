#!/bin/bash
# ncu --set full of the guide-mode LT sampler (cfg4) at the bench batch and at 1M sets.
mkdir -p gpurun_out
NCU="ncu --set full --import-source on --clock-control none -s 1 -c 1"
run() {  # name kernel-regex command...
  local name=$1 kr=$2; shift 2
  timeout 300 "$@" > gpurun_out/$name.log 2>&1 && \
    timeout 900 $NCU -k regex:$kr -o gpurun_out/$name -f "$@" > gpurun_out/$name.ncu.log 2>&1
  echo "$name rc=$?"; tail -1 gpurun_out/$name.log
}
#run g_cfg4_65k k_sample_lt_guide python tools/profile_sampler.py cfg4 --sets 65536 --lt-scan 2
run g_cfg4_1m k_sample_lt_guide python tools/profile_sampler.py cfg4 --sets 1048576 --lt-scan 2
