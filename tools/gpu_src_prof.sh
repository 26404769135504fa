# ncu --set full --import-source of the hot kernels of one steady-state op (run under gpurun);
# the report comes back as gpurun_out/<tag>.ncu-rep (read it here with ncu -i ... --page source)
# usage: bash tools/gpu_src_prof.sh TAG C4 dilate 16 [kernel regex]
tag=$1; cfg=$2; op=$3; r=$4; kre=${5:-"p1[gs]_kernel|levels_kernel|pass2s_kernel"}
timeout 300 python tools/run_op.py $cfg $op $r 1 > gpurun_out/${tag}_runop.log 2>&1 || exit 1
PROFILE_LAST=1 timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off \
  -k regex:"$kre" -c 12 -o gpurun_out/${tag} python tools/run_op.py $cfg $op $r 3 > gpurun_out/${tag}_ncu.log 2>&1
ls -la gpurun_out/${tag}.ncu-rep
