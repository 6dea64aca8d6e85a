#!/bin/bash
mkdir -p gpurun_out
A="cfg5 --n 300000 --m 11000000 --sets 8192"
timeout 200 python tools/profile_sampler.py $A --ic-mode 3 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sample_ic_cta -s 1 -c 1 \
  -o gpurun_out/cta2_cfg5s -f python tools/profile_sampler.py $A --ic-mode 3 > gpurun_out/cta2_ncu.log 2>&1
tail -2 gpurun_out/cta2_ncu.log
