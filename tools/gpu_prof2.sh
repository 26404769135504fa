# bench (C5 default) + one C5 op under ncu --set full for all pass-1 / levels launches
tag=${1:-p5}
python bench.py --steps 3 --warmup 3 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
python tools/run_op.py C5 shell 16 1 > gpurun_out/${tag}_runop.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"p1_kernel|levels_kernel" -c 60 -o gpurun_out/${tag}_full python tools/run_op.py C5 shell 16 1 > gpurun_out/${tag}_ncu.log 2>&1
