# final check of the tree with the host pipeline (run under gpurun): all GPU tests, smoke, the default
# bench line + reference arm, e2e lines of the workloads the library splits, the ncu launch list of the
# default command.  usage: bash tools/gpu_round_check.sh TAG
tag=${1:-pipe4}
DEXEL_PARITY_REPORT=gpurun_out/${tag}_parity.json timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/${tag}_smoke.log 2>&1
python bench.py --steps 5 --warmup 3 > gpurun_out/${tag}_bench_c5.json 2> gpurun_out/${tag}_bench_c5.err
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${tag}_bench_reference.json 2> gpurun_out/${tag}_bench_reference.err
: > gpurun_out/${tag}_e2e.jsonl
for a in "C4 dilate 8" "C4 dilate 16" "C4 dilate 32" "C3 dilate 8" "C3 erode 8" "C4 dilate 4"; do
  set -- $a
  timeout 600 python bench.py --config $1 --op $2 --r $3 --steps 10 --warmup 3 --no-cpu \
    >> gpurun_out/${tag}_e2e.jsonl 2>> gpurun_out/${tag}_e2e.err
done
python tools/e2e_table.py gpurun_out/${tag}_e2e.jsonl > gpurun_out/${tag}_e2e_summary.txt
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/${tag}_launches.log 2>&1
echo done
