# The streamed host-to-host op (dexel_pipe_run) on the GPU box: its tests, then the e2e number of
# the headline workload for several slab counts (and two smaller configs).  usage: bash tools/gpu_pipe.sh TAG
tag=${1:-pipe}
timeout 900 python -m pytest tests/test_gpu_pipe.py -q -x > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
: > gpurun_out/${tag}_e2e.jsonl
for s in 2 4 8 16 32; do
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --e2e-slabs $s >> gpurun_out/${tag}_e2e.jsonl 2>> gpurun_out/${tag}_e2e.err
done
for a in "C4 dilate 16" "C4 dilate 64" "C3 dilate 8" "C2 shell 4"; do
  set -- $a
  for s in 4 8; do
    timeout 600 python bench.py --config $1 --op $2 --r $3 --steps 5 --warmup 3 --no-cpu --e2e-slabs $s \
      >> gpurun_out/${tag}_e2e.jsonl 2>> gpurun_out/${tag}_e2e.err
  done
done
python tools/e2e_table.py gpurun_out/${tag}_e2e.jsonl > gpurun_out/${tag}_e2e_summary.txt
echo done
