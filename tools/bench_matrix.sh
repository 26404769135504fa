# The BASELINE.json measurement matrix (run under gpurun): one bench.py line per (config, op, r),
# each with its cpu_baseline (BASELINE.md section 3 sample), into gpurun_out/<tag>_matrix.jsonl
# usage: bash tools/bench_matrix.sh TAG [steps]
tag=${1:-matrix}; steps=${2:-10}
out=gpurun_out/${tag}_matrix.jsonl
: > $out
for a in "C1 dilate 3" "C1 erode 3" "C2 dilate 4" "C2 erode 4" "C2 shell 4" "C3 dilate 8" "C3 erode 8" \
         "C4 dilate 1" "C4 dilate 2" "C4 dilate 4" "C4 dilate 8" "C4 dilate 16" "C4 dilate 32" "C4 dilate 64" \
         "C5 shell 16"; do
  set -- $a
  timeout 900 python bench.py --config $1 --op $2 --r $3 --steps $steps --warmup 3 >> $out 2>> gpurun_out/${tag}_matrix.err
done
echo done
