#!/bin/bash
# A/B of the IC sampler: build_cmp/librrgpu_old.so vs the in-tree library.
for c in "cfg1 --sets 65536 --ic-mode 2" "cfg3 --sets 1048576" "cfg5 --n 300000 --m 11000000 --sets 8192 --ic-mode 2" "cfg5 --n 300000 --m 11000000 --sets 8192 --ic-mode 3" "cfg5 --sets 32768"; do
  RRGPU_LIB=build_cmp/librrgpu_old.so timeout 120 python tools/profile_sampler.py $c | tail -1 | sed 's/^/old /'
  timeout 120 python tools/profile_sampler.py $c | tail -1 | sed 's/^/new /'
done
