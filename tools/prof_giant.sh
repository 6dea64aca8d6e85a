#!/bin/bash
# ncu source-level capture of the block schedule on cfg3's largest IMM-size set
# (slot 46726 of a 65,536-set batch, 35.6K members, 833K inspected in-edges).
mkdir -p gpurun_out
timeout 200 python tools/one_slot.py cfg3 46726 3 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_sample_ic_cta -s 1 -c 1 \
  -o gpurun_out/giant_cfg3 -f python tools/one_slot.py cfg3 46726 3 > gpurun_out/giant_ncu.log 2>&1
tail -2 gpurun_out/giant_ncu.log
