mkdir -p gpurun_out
timeout 1200 python -m pytest tests/ -q -m gpu > gpurun_out/final_tests.log 2>&1; tail -1 gpurun_out/final_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python tools/imm_table.py > gpurun_out/imm_table_r1h.jsonl 2> gpurun_out/imm_table.err; echo imm rc=$?
timeout 900 python bench.py > gpurun_out/bench_r1o.json 2> gpurun_out/bench.err; echo bench rc=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r1o.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_bench.log 2>&1; echo ncu rc=$?
