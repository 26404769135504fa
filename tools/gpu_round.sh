# round profile (run under gpurun): C5 bench line, reference arm, C4/C3 bench lines, the ncu launch list of
# the bench command, and one ncu --set full capture of every pass1/levels/pass2 launch of one C5 shell op
tag=${1:-r01}
python bench.py --steps 5 --warmup 3 > gpurun_out/${tag}_bench_c5.json 2> gpurun_out/${tag}_bench_c5.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${tag}_bench_reference.json 2> gpurun_out/${tag}_bench_reference.err
: > gpurun_out/${tag}_bench_c4c3.jsonl
for a in "C4 dilate 1" "C4 dilate 4" "C4 dilate 16" "C4 dilate 64" "C3 dilate 8" "C2 shell 4" \
         "C4 dilate_slices 16" "C5 shell_slices 16" "C3 erode_slices 8"; do
  set -- $a
  timeout 600 python bench.py --config $1 --op $2 --r $3 --steps 5 --warmup 3 --no-cpu >> gpurun_out/${tag}_bench_c4c3.jsonl 2>> gpurun_out/${tag}_bench_c4c3.err
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/${tag}_launches.log 2>&1
python tools/run_op.py C5 shell 16 1 > gpurun_out/${tag}_runop.log 2>&1 && \
PROFILE_LAST=1 ncu --set full --clock-control none --profile-from-start off \
  -k regex:"p1_kernel|p1_dual_kernel|levels_kernel|pass2s_kernel" -c 60 \
  -o /tmp/${tag}_full python tools/run_op.py C5 shell 16 3 > gpurun_out/${tag}_ncu.log 2>&1
echo "done rc=$?" >> gpurun_out/${tag}_ncu.log
# the report itself stays on the box (tens of MB): bring back its raw page and the summaries
ncu -i /tmp/${tag}_full.ncu-rep --page raw --csv > /tmp/${tag}_raw.csv
python tools/ncu_summary.py /tmp/${tag}_raw.csv "${tag} C5 shell r=16, one op, ncu --set full" > gpurun_out/${tag}_ncu_full_summary.txt 2>&1
cp profiles/traffic.json gpurun_out/${tag}_traffic.json
python tools/ncu_traffic.py /tmp/${tag}_raw.csv C5:shell:16.0 gpurun_out/${tag}_traffic.json > gpurun_out/${tag}_traffic.log 2>&1
gzip -c /tmp/${tag}_raw.csv > gpurun_out/${tag}_ncu_raw.csv.gz
