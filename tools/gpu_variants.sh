# A/B of library variants built into exp/libdexel_<name>.so (run under gpurun): the quick parity
# subset with each, then per-op timings.  usage: bash tools/gpu_variants.sh TAG "v0 v1 v2" "C5 shell 16" ...
tag=$1; vars=$2; shift 2
work=("$@")
cp paper_1804_08968_b200/libdexel.so /tmp/libdexel_orig.so
for v in $vars; do
  cp exp/libdexel_$v.so paper_1804_08968_b200/libdexel.so
  touch paper_1804_08968_b200/libdexel.so
  timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "ops_random or configs_all or edge or fused or capacity or many" \
    > gpurun_out/${tag}_${v}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_${v}_pytest.log
  for a in "${work[@]}"; do timeout 300 python tools/time_op.py $a 3; done > gpurun_out/${tag}_${v}_times.log 2>&1
done
cp /tmp/libdexel_orig.so paper_1804_08968_b200/libdexel.so
echo done
