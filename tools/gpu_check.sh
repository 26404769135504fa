# usage: bash tools/gpu_check.sh [tag]  -- GPU tests + per-op timing matrix (run under gpurun)
tag=${1:-chk}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
( for r in 1 4 16 64; do timeout 300 python tools/time_op.py C4 dilate $r 3; done
  timeout 300 python tools/time_op.py C3 dilate 8 3
  timeout 300 python tools/time_op.py C2 shell 4 5
  timeout 300 python tools/time_op.py C5 shell 16 3 ) > gpurun_out/${tag}_times.log 2>&1
