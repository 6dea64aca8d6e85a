#!/bin/bash
# Round-end evidence: bench launch list + ncu --set full of the dominant kernels.
# Every ncu command runs only after the same command exited 0 without ncu.
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-imm --no-cpu-baseline"
timeout 300 $B > gpurun_out/fb_plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_bench.csv $B > gpurun_out/fb_ncu.log 2>&1
echo "launch list rc=$?"
NCU="ncu --set full --import-source on --clock-control none -s 1 -c 1"
run() {  # name kernel-regex command...
  local name=$1 kr=$2; shift 2
  timeout 300 "$@" > gpurun_out/$name.log 2>&1 && \
    timeout 600 $NCU -k regex:$kr -o gpurun_out/$name -f "$@" > gpurun_out/$name.ncu.log 2>&1
  echo "$name rc=$?"; tail -1 gpurun_out/$name.log
}
run fin_cfg4_bsearch k_sample_lt python tools/profile_sampler.py cfg4 --sets 65536 --lt-scan 1
run fin_cfg4_linear k_sample_lt python tools/profile_sampler.py cfg4 --sets 65536 --lt-scan 0
run fin_cfg1_warp k_sample_ic_warp python tools/profile_sampler.py cfg1 --sets 65536 --ic-mode 2
run fin_cfg3_lane k_sample_ic python tools/profile_sampler.py cfg3 --sets 262144 --ic-mode 1
