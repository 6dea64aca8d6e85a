python -m pytest tests/test_gpu_sampling.py tests/test_gpu_imm.py tests/test_gpu_selection.py tests/test_gpu_checked.py -x -q 2>&1 | tail -3
python tools/imm_gpu.py cfg1 cfg2 cfg3 cfg4 cfg5 2>&1 | grep imm
for c in cfg1 cfg3 cfg5; do python tools/e2e_imm_parts.py $c 2>&1 | head -3; done
