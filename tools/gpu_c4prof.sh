# ncu --set full of every pass1/levels/pass2 launch of one steady-state op, per (config, op, r)
# (run under gpurun): summaries + traffic into gpurun_out/<tag>_*
# usage: bash tools/gpu_c4prof.sh TAG "C4 dilate 1" "C4 dilate 16" ...
tag=$1; shift
for a in "$@"; do
  set -- $a
  name="${1}_${2}_${3}"
  timeout 300 python tools/run_op.py $1 $2 $3 1 > gpurun_out/${tag}_${name}_runop.log 2>&1 || continue
  PROFILE_LAST=1 timeout 900 ncu --set full --clock-control none --profile-from-start off \
    -k regex:"p1[gs]_kernel|levels_kernel|pass2s_kernel" -c 60 \
    -f -o /tmp/${tag}_${name} python tools/run_op.py $1 $2 $3 3 > gpurun_out/${tag}_${name}_ncu.log 2>&1
  ncu -i /tmp/${tag}_${name}.ncu-rep --page raw --csv > /tmp/${tag}_${name}_raw.csv
  python tools/ncu_summary.py /tmp/${tag}_${name}_raw.csv "${tag} $1 $2 r=$3, one op, ncu --set full" \
    > gpurun_out/${tag}_${name}_ncu_summary.txt 2>&1
  python tools/ncu_traffic.py /tmp/${tag}_${name}_raw.csv "$1:$2:$3.0" gpurun_out/${tag}_traffic.json \
    > gpurun_out/${tag}_${name}_traffic.log 2>&1
done
echo done
