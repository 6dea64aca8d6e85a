#!/bin/bash
# IC sampler sweep on the GPU box: schedule (lane/warp/auto) x config.
for cfg in ${CFGS:-"cfg1 --sets 65536" "cfg1 --sets 1048576" "cfg3 --sets 65536" "cfg3 --sets 262144" "cfg3 --sets 1048576" "cfg5 --n 300000 --m 11000000 --sets 8192" "cfg5 --sets 32768"}; do
  for mode in ${IC_MODES:-1 2 0}; do
    timeout ${TMO:-120} python tools/profile_sampler.py $cfg --ic-mode $mode || echo "FAILED/TIMEOUT rc=$? $cfg mode $mode"
  done
done
