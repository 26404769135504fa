# bench (C5 default) + launch list + ncu --set full of every launch of the dominant kernel in one op
k=${1:-levels_kernel}; tag=${2:-p1}
python bench.py --steps 3 --warmup 3 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
python tools/run_op.py C5 shell 16 1 > gpurun_out/${tag}_runop.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$k" -c 40 -o gpurun_out/${tag}_full python tools/run_op.py C5 shell 16 1 > gpurun_out/${tag}_ncu.log 2>&1
