#!/bin/bash
mkdir -p gpurun_out
A="cfg4 --sets ${SETS:-8192} --lt-scan 1"
timeout 200 python tools/profile_sampler.py $A && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sample_lt -s 1 -c 1 \
  -o gpurun_out/lt_${SETS:-8192} -f python tools/profile_sampler.py $A > gpurun_out/lt_ncu.log 2>&1
tail -2 gpurun_out/lt_ncu.log
