# e2e through the suggested slab count for the matrix's larger workloads + the default bench line
# (run under gpurun).  usage: bash tools/gpu_pipe2.sh TAG
tag=${1:-pipe2}
timeout 900 python -m pytest tests/test_gpu_pipe.py tests/test_gpu_slabs.py -q -x > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
python bench.py --steps 5 --warmup 3 > gpurun_out/${tag}_bench_c5.json 2> gpurun_out/${tag}_bench_c5.err
: > gpurun_out/${tag}_e2e.jsonl
for a in "C4 dilate 1" "C4 dilate 2" "C4 dilate 4" "C4 dilate 8" "C4 dilate 16" "C4 dilate 32" "C3 dilate 8" "C3 erode 8"; do
  set -- $a
  timeout 600 python bench.py --config $1 --op $2 --r $3 --steps 10 --warmup 3 --no-cpu \
    >> gpurun_out/${tag}_e2e.jsonl 2>> gpurun_out/${tag}_e2e.err
done
for s in 2 3; do
  timeout 600 python bench.py --config C4 --op dilate --r 64 --steps 5 --warmup 3 --no-cpu --e2e-slabs $s \
    >> gpurun_out/${tag}_e2e.jsonl 2>> gpurun_out/${tag}_e2e.err
done
python tools/e2e_table.py gpurun_out/${tag}_e2e.jsonl > gpurun_out/${tag}_e2e_summary.txt
DEXEL_DEBUG=1 timeout 300 python bench.py --config C2 --op shell --r 4 --steps 3 --warmup 3 --no-cpu --e2e-slabs 8 \
  > gpurun_out/${tag}_c2_dbg.json 2> gpurun_out/${tag}_c2_dbg.err
echo done
