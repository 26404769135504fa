# Round measurement (run under gpurun): GPU tests, smoke, ncu --set full of every pass1/levels/pass2
# launch of one op per workload (summaries + DRAM traffic -> the bench lines' roofline.traffic), the
# default bench line + reference arm, the BASELINE.json matrix (each line with its cpu_baseline),
# the ncu launch list of the default bench command, and --gpus 2 on a 1-GPU box (must fail loudly).
# usage: bash tools/gpu_final.sh TAG [matrix steps]
tag=${1:-final}; steps=${2:-10}
DEXEL_PARITY_REPORT=gpurun_out/${tag}_parity.json timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/${tag}_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/${tag}_smoke.log
cp profiles/traffic.json gpurun_out/${tag}_traffic.json
bash tools/gpu_c4prof.sh $tag "C5 shell 16" "C4 dilate 1" "C4 dilate 4" "C4 dilate 16" "C4 dilate 64" "C3 dilate 8" \
  "C3 erode 8" "C2 shell 4" > gpurun_out/${tag}_prof.log 2>&1
# complete per-op DRAM traffic from a light ncu pass (the --set full capture of the big ops stops early)
bash tools/gpu_traffic.sh $tag "C5 shell 16" "C4 dilate 64" "C4 dilate 32" "C4 dilate 16" "C4 dilate 8" "C4 dilate 4" \
  "C4 dilate 2" "C4 dilate 1" "C3 dilate 8" "C3 erode 8" "C2 dilate 4" "C2 erode 4" "C2 shell 4" > gpurun_out/${tag}_traffic_run.log 2>&1
cp gpurun_out/${tag}_traffic.json profiles/traffic.json   # (this box's copy: the bench lines below read it)
python bench.py --steps 5 --warmup 3 > gpurun_out/${tag}_bench_c5.json 2> gpurun_out/${tag}_bench_c5.err
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${tag}_bench_reference.json \
  2> gpurun_out/${tag}_bench_reference.err
bash tools/bench_matrix.sh $tag $steps
# GPU dexelisation lines: shapes (C2, C4, C5) and the noisy gyroid (C3)
for c in C2 C3 C4 C5; do timeout 900 python bench.py --config $c --op rasterize --steps 5 --warmup 3; done \
  > gpurun_out/${tag}_raster.jsonl 2> gpurun_out/${tag}_raster.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/${tag}_launches.log 2>&1
timeout 300 python bench.py --gpus 2 --steps 2 --warmup 3 > gpurun_out/${tag}_gpus2.log 2>&1
echo "gpus2 rc=$?" >> gpurun_out/${tag}_gpus2.log
echo done
