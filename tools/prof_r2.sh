#!/bin/bash
# Round-2 evidence: launch list of the headline bench + ncu --set full of the
# dominant kernels of each measured block. Each ncu command runs only after the
# same command exited 0 without ncu. Output: gpurun_out/r2_*.ncu-rep
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-imm --no-cpu-baseline --no-extra --small-sets 0 --linear-sets 0 --sharded-imm 0"
timeout 300 $B > gpurun_out/r2_lb_plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r2_launches_bench.csv $B > gpurun_out/r2_lb_ncu.log 2>&1
echo "launch list rc=$?"
NCU="ncu --set full --import-source on --clock-control none -s 1 -c 1"
run() {  # name kernel-regex command...
  local name=$1 kr=$2; shift 2
  timeout 300 "$@" > gpurun_out/$name.log 2>&1 && \
    timeout 900 $NCU -k regex:$kr -o gpurun_out/$name -f "$@" > gpurun_out/$name.ncu.log 2>&1
  echo "$name rc=$?"; tail -1 gpurun_out/$name.log
}
run r2_ic_cfg1_1m k_sample_ic python tools/profile_sampler.py cfg1 --sets 1048576
run r2_ic_cfg5_32k k_sample_ic python tools/profile_sampler.py cfg5 --sets 32768
run r2_giant_cfg3c k_sample_ic_cta python tools/profile_sampler.py cfg3c --sets 2048 --ic-mode 3
run r2_select_cluster_cfg2 k_select_cluster python tools/profile_select.py cfg2 --sets 8192 --repeat 2
run r2_select_dense_cfg3c k_select python tools/profile_select.py cfg3c --sets 4096 --repeat 2
run r2_guide_cfg4_1m k_sample_lt_guide python tools/profile_sampler.py cfg4 --sets 1048576 --lt-scan 2
