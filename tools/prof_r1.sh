set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py > gpurun_out/bench_r1b.json 2> gpurun_out/bench_r1b.err; cat gpurun_out/bench_r1b.json
P1="python tools/profile_sampler.py cfg1 --sets 65536"
P2="python tools/profile_sampler.py cfg4 --sets 65536 --lt-scan 1"
P3="python tools/profile_sampler.py cfg4 --sets 65536 --lt-scan 0"
P4="python tools/profile_sampler.py cfg5 --n 300000 --m 11000000 --sets 8192"
NCU="ncu --set full --import-source on --clock-control none -k regex:k_sample -s 1 -c 1"
$P1 > gpurun_out/p1.log 2>&1 && $NCU -o gpurun_out/prof_cfg1_ic $P1 > gpurun_out/ncu1.log 2>&1; cat gpurun_out/p1.log
$P2 > gpurun_out/p2.log 2>&1 && $NCU -o gpurun_out/prof_cfg4_bsearch $P2 > gpurun_out/ncu2.log 2>&1; cat gpurun_out/p2.log
$P3 > gpurun_out/p3.log 2>&1 && $NCU -o gpurun_out/prof_cfg4_linear $P3 > gpurun_out/ncu3.log 2>&1; cat gpurun_out/p3.log
$P4 > gpurun_out/p4.log 2>&1 && $NCU -o gpurun_out/prof_cfg5s_ic $P4 > gpurun_out/ncu4.log 2>&1; cat gpurun_out/p4.log
B="python bench.py --steps 2 --warmup 1 --e2e-steps 1 --no-imm"
$B > gpurun_out/bench_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv $B > gpurun_out/ncu_bench.log 2>&1
ls -la gpurun_out
