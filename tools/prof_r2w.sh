#!/bin/bash
# Late round-2 evidence (after the code-size and K0 changes): stability sweep, the
# launch list of the headline bench, ncu --set full of the IC warp schedule (cfg1),
# of the guide walk (cfg4) and of the hub CDF scan. Each ncu command runs only
# after the same command exited 0 without ncu. Output: gpurun_out/r2w_*
mkdir -p gpurun_out
PASSES=1 bash tools/stress.sh > gpurun_out/r2w_stress.log 2>&1
grep -c "rc=0" gpurun_out/r2w_stress.log; grep -v "rc=0" gpurun_out/r2w_stress.log
B="python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-imm --no-cpu-baseline --no-extra --small-sets 0 --linear-sets 0 --sharded-imm 0"
timeout 300 $B > gpurun_out/r2w_lb_plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r2w_launches_bench.csv $B > gpurun_out/r2w_lb_ncu.log 2>&1
echo "launch list rc=$?"
NCU="ncu --set full --import-source on --clock-control none -s 1 -c 1"
run() {  # name kernel-regex command...
  local name=$1 kr=$2; shift 2
  timeout 300 "$@" > gpurun_out/$name.log 2>&1 && \
    timeout 900 $NCU -k regex:$kr -o gpurun_out/$name -f "$@" > gpurun_out/$name.ncu.log 2>&1
  echo "$name rc=$?"; tail -1 gpurun_out/$name.log
}
run r2w_ic_cfg1_1m k_sample_ic python tools/profile_sampler.py cfg1 --sets 1048576
run r2w_guide_cfg4_1m k_sample_lt_guide python tools/profile_sampler.py cfg4 --sets 1048576 --lt-scan 2
timeout 300 python tools/profile_sampler.py cfg4 --sets 4096 --lt-scan 2 > gpurun_out/r2w_cdf.log 2>&1 && \
  timeout 900 ncu --set full --import-source on --clock-control none -c 1 -k regex:k_build_cdf_long \
    -o gpurun_out/r2w_cdf_long_cfg4 -f python tools/profile_sampler.py cfg4 --sets 4096 --lt-scan 2 > gpurun_out/r2w_cdf.ncu.log 2>&1
echo "cdf rc=$?"
