#!/bin/bash
# Round-1 profiling pass 2: ncu full captures of the samplers after the
# cooperative-expansion/jump-table changes + IMM launch list + LT arity sweep.
NCU="ncu --set full --import-source on --clock-control none -k regex:k_sample -s 1 -c 1"
P1="python tools/profile_sampler.py cfg5 --n 300000 --m 11000000 --sets 8192 --ic-coop-min 256"
P2="python tools/profile_sampler.py cfg1 --sets 65536 --ic-coop-min 256"
P3="python tools/profile_sampler.py cfg4 --sets 65536 --lt-scan 1 --lt-kary 16"
for k in 2 4 8 16; do python tools/profile_sampler.py cfg4 --sets 65536 --lt-scan 1 --lt-kary $k; done
for k in 2 16; do python tools/profile_sampler.py cfg2 --sets 1048576 --lt-scan 1 --lt-kary $k; done
python tools/profile_sampler.py cfg4 --sets 65536 --lt-scan 0
$P1 > gpurun_out/q1.log 2>&1 && $NCU -o gpurun_out/prof2_cfg5s_ic $P1 > gpurun_out/nq1.log 2>&1; cat gpurun_out/q1.log
$P2 > gpurun_out/q2.log 2>&1 && $NCU -o gpurun_out/prof2_cfg1_ic $P2 > gpurun_out/nq2.log 2>&1; cat gpurun_out/q2.log
$P3 > gpurun_out/q3.log 2>&1 && $NCU -o gpurun_out/prof2_cfg4_kary16 $P3 > gpurun_out/nq3.log 2>&1; cat gpurun_out/q3.log
I="python tools/profile_imm.py cfg4 --repeat 2"
$I > gpurun_out/imm_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_imm_cfg4.csv $I > gpurun_out/nq4.log 2>&1; cat gpurun_out/imm_plain.log
