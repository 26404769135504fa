tag=${1:-m5}
( for ch in 12 17; do
    export DEXEL_LV_CHUNK=$ch; echo "== chunk $ch"
    for r in 4 16 64; do timeout 300 python tools/time_op.py C4 dilate $r 3; done
    timeout 300 python tools/time_op.py C5 shell 16 2
  done ) > gpurun_out/${tag}_times.log 2>&1
unset DEXEL_LV_CHUNK
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest.log
