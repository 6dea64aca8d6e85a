#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_selection.py tests/test_gpu_imm.py -x -q 2>&1 | tail -3
timeout 900 python tools/imm_table.py > gpurun_out/imm_table.jsonl 2> gpurun_out/imm_table.err; echo imm_table rc=$?
