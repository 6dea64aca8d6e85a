#!/bin/bash
P1="python tools/profile_sampler.py cfg3 --sets 262144 --ic-mode 2"
$P1 > gpurun_out/x1.log 2>&1 && ncu --set full --import-source on --clock-control none -k regex:k_sample_ic_warp -s 3 -c 1 -o gpurun_out/prof4_cfg3_wide $P1 > gpurun_out/nx1.log 2>&1; cat gpurun_out/x1.log; tail -3 gpurun_out/nx1.log
