#!/bin/bash
P1="python tools/profile_sampler.py cfg5 --n 300000 --m 11000000 --sets 8192 --ic-mode 2"
$P1 > gpurun_out/w1.log 2>&1 && ncu --set full --import-source on --clock-control none -k regex:k_sample_ic_warp -s 1 -c 1 -o gpurun_out/prof3_cfg5s_warp $P1 > gpurun_out/nw1.log 2>&1; cat gpurun_out/w1.log
