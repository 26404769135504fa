# DRAM traffic of every pass1/levels/pass2 launch of one steady-state op (run under gpurun): a
# light ncu pass (dram bytes + duration only: big ops replay without the --set full save/restore
# of their memory) -> gpurun_out/<tag>_traffic.json.  usage: bash tools/gpu_traffic.sh TAG "C5 shell 16" ...
tag=$1; shift
for a in "$@"; do
  set -- $a
  n=${1}_${2}_${3}
  PROFILE_LAST=1 timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none --profile-from-start off -k regex:"p1[gs]_kernel|levels_kernel|pass2s_kernel" \
    -f -o /tmp/${tag}_light_${n} python tools/run_op.py $1 $2 $3 3 > gpurun_out/${tag}_${n}_traffic_ncu.log 2>&1
  ncu -i /tmp/${tag}_light_${n}.ncu-rep --page raw --csv > /tmp/${tag}_light_${n}_raw.csv
  python tools/ncu_traffic.py /tmp/${tag}_light_${n}_raw.csv "$1:$2:$3.0" gpurun_out/${tag}_traffic.json \
    > gpurun_out/${tag}_${n}_traffic.log 2>&1
done
echo done
