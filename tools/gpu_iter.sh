# one iteration (run under gpurun): GPU parity suite (or a -k subset), then per-op timings
# usage: bash tools/gpu_iter.sh TAG "pytest -k expr or ''" "C5 shell 16" "C4 dilate 64" ...
tag=$1; kexpr=$2; shift 2
if [ -n "$kexpr" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -k "$kexpr" > gpurun_out/${tag}_pytest.log 2>&1
else
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1
fi
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
for a in "$@"; do timeout 300 python tools/time_op.py $a 3; done > gpurun_out/${tag}_times.log 2>&1
echo done
