#!/bin/bash
# IC sampler sweep on the GPU box: cooperative-expansion threshold x config.
set -x
for cfg in "cfg1 --sets 65536" "cfg1 --sets 1048576" "cfg3 --sets 1048576" "cfg5 --n 300000 --m 11000000 --sets 8192" "cfg5 --sets 32768"; do
  for cm in 4294967295 1024 256 64; do
    timeout 300 python tools/profile_sampler.py $cfg --ic-coop-min $cm
  done
done
