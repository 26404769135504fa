# usage: bash tools/gpu_modes.sh tag -- A/B the level-set kernel variants (run under gpurun)
tag=${1:-modes}
( for m in columns lanes; do
    export DEXEL_LEVELS=$m
    for r in 4 8 16 32 64; do timeout 300 python tools/time_op.py C4 dilate $r 3; done
    timeout 300 python tools/time_op.py C3 dilate 8 3
    timeout 300 python tools/time_op.py C5 shell 16 2
  done ) > gpurun_out/${tag}_times.log 2>&1
unset DEXEL_LEVELS
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest.log
