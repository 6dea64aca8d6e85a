#!/bin/bash
# IC sampler sweep on the GPU box: library variant x cooperative threshold x config.
for lib in paper_2411_09473_b200/librrgpu.so paper_2411_09473_b200/librrgpu_mb2.so; do
  [ -f $lib ] || continue
  echo "== $lib"
  for cfg in "cfg1 --sets 65536" "cfg1 --sets 1048576" "cfg3 --sets 1048576" "cfg5 --n 300000 --m 11000000 --sets 8192" "cfg5 --sets 32768"; do
    for cm in ${COOP_MINS:-4294967295 1024 256}; do
      RRGPU_LIB=$lib timeout 300 python tools/profile_sampler.py $cfg --ic-coop-min $cm
    done
  done
done
