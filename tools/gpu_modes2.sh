tag=${1:-m2}
( for cfg in "columns 17" "columns 12" "columns 9" "lanes 17"; do
    set -- $cfg; export DEXEL_LEVELS=$1 DEXEL_LV_CHUNK=$2; echo "== $cfg"
    for r in 4 16 64; do timeout 300 python tools/time_op.py C4 dilate $r 3; done
    timeout 300 python tools/time_op.py C5 shell 16 2
  done ) > gpurun_out/${tag}_times.log 2>&1
unset DEXEL_LEVELS DEXEL_LV_CHUNK
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest.log
