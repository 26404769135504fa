# ncu --set full (with source) of the first levels_kernel launch of one C5 shell op
tag=${1:-lv}
python tools/run_op.py C5 shell 16 1 > gpurun_out/${tag}_runop.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"${2:-levels_kernel}" -c 1 -o gpurun_out/${tag}_full python tools/run_op.py C5 shell 16 1 > gpurun_out/${tag}_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_ncu.log
