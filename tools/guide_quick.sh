mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sampling.py -x -q -k "guide or trip" > gpurun_out/g1_tests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/g1_tests.log
for sc in "1 0" "2 1" "2 2" "2 4"; do set -- $sc; timeout 300 python tools/profile_sampler.py cfg4 --sets 65536 --lt-scan $1 --lt-guide-mult $2 2>&1 | tail -2; done
for sc in "1 0" "2 2"; do set -- $sc; timeout 300 python tools/profile_sampler.py cfg2 --sets 1048576 --lt-scan $1 --lt-guide-mult $2 2>&1 | tail -2; done
timeout 300 python tools/profile_sampler.py cfg4 --sets 1048576 --lt-scan 2 2>&1 | tail -1
timeout 300 python tools/profile_sampler.py cfg4 --sets 1048576 --lt-scan 1 2>&1 | tail -1
