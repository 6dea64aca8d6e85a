#!/bin/bash
# ncu --set full of the block IC schedule on a full-size cfg5 batch (8,192 sets):
# is the whole-list expansion L2-bound on the per-lane jump-table reads?
mkdir -p gpurun_out
A="cfg5 --sets 8192 --ic-mode 3"
timeout 200 python tools/profile_sampler.py $A && \
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_sample_ic_cta -s 1 -c 1 \
  -o gpurun_out/cta_cfg5_full -f python tools/profile_sampler.py $A > gpurun_out/cta_cfg5_ncu.log 2>&1
tail -2 gpurun_out/cta_cfg5_ncu.log
