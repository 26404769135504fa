tag=${1:-m6}
( for ch in 12 17; do
    export DEXEL_LV_CHUNK=$ch; echo "== chunk $ch"
    for r in 8 16 32; do timeout 300 python tools/time_op.py C4 dilate $r 3; done
    timeout 300 python tools/time_op.py C5 shell 16 2
  done ) > gpurun_out/${tag}_times.log 2>&1
