#!/bin/bash
mkdir -p gpurun_out
A="cfg5 --n 300000 --m 11000000 --sets 8192 --ic-mode 2"
timeout 200 python tools/profile_sampler.py $A && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sample_ic_warp -s 1 -c 1 \
  -o gpurun_out/warp_cfg5s -f python tools/profile_sampler.py $A > gpurun_out/warp5_ncu.log 2>&1
tail -2 gpurun_out/warp5_ncu.log
