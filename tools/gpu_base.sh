# Baseline check of HEAD (run under gpurun): full GPU suite, smoke, per-op timings, default bench line
# usage: bash tools/gpu_base.sh TAG
tag=${1:-base}
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${tag}_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/${tag}_smoke.log
( for r in 1 4 16 64; do timeout 300 python tools/time_op.py C4 dilate $r 3; done
  timeout 300 python tools/time_op.py C3 dilate 8 3
  timeout 300 python tools/time_op.py C2 shell 4 5
  timeout 300 python tools/time_op.py C5 shell 16 3 ) > gpurun_out/${tag}_times.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/${tag}_bench_c5.json 2> gpurun_out/${tag}_bench_c5.err
echo done
