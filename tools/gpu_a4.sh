timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/a4_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/a4_pytest.log
for a in "C1 dilate 3" "C1 erode 3" "C2 dilate 4" "C2 shell 4" "C3 dilate 8" "C4 dilate 1" "C4 dilate 16" "C5 shell 16"; do timeout 300 python tools/time_op.py $a 5; done > gpurun_out/a4_times.log 2>&1
DEXEL_DEBUG=1 timeout 300 python tools/time_op.py C5 shell 16 1 > gpurun_out/a4_debug_c5.log 2>&1
DEXEL_DEBUG=1 timeout 300 python tools/time_op.py C4 dilate 16 1 > gpurun_out/a4_debug_c4.log 2>&1
