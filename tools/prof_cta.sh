#!/bin/bash
# IC schedule sweep (lane / warp / block / auto) and one ncu capture of the block kernel.
mkdir -p gpurun_out
CFGS="cfg1 --sets 65536|cfg1 --sets 1048576|cfg3 --sets 65536|cfg3 --sets 1048576|cfg5 --n 300000 --m 11000000 --sets 8192|cfg5 --sets 32768" \
IC_MODES="${IC_MODES:-1 2 3 0}"
IFS="|"; for c in $CFGS; do IFS=" "; for mode in $IC_MODES; do
  timeout 150 python tools/profile_sampler.py $c --ic-mode $mode 2>&1 | tail -1; done; done
if [ -n "$NCU" ]; then
  timeout 200 python tools/profile_sampler.py cfg5 --n 300000 --m 11000000 --sets 8192 --ic-mode 3 && \
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sample_ic_cta -s 1 -c 1 \
    -o gpurun_out/cta_cfg5s -f python tools/profile_sampler.py cfg5 --n 300000 --m 11000000 --sets 8192 --ic-mode 3 > gpurun_out/cta_ncu.log 2>&1
  tail -3 gpurun_out/cta_ncu.log
fi
