# quick GPU check (run under gpurun): parity subset, then per-op timings
# usage: bash tools/gpu_quick.sh TAG [pytest -k expression]
tag=${1:-q}; kexpr=${2:-"pass1 or ops_random or configs_all or edge or fused or capacity or many or slabs or loopback"}
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py -m gpu -x -q -k "$kexpr" > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
( for r in 1 2 4 8 16 64; do timeout 300 python tools/time_op.py C4 dilate $r 3; done
  timeout 300 python tools/time_op.py C3 dilate 8 3
  timeout 300 python tools/time_op.py C3 erode 8 3
  timeout 300 python tools/time_op.py C2 shell 4 5
  timeout 300 python tools/time_op.py C5 shell 16 3 ) > gpurun_out/${tag}_times.log 2>&1
echo done
