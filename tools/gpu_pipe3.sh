tag=${1:-pipe3}
for a in "C2 shell 4 8" "C3 erode 8 2" "C4 dilate 1 4"; do
  set -- $a
  DEXEL_DEBUG=1 timeout 300 python bench.py --config $1 --op $2 --r $3 --steps 3 --warmup 3 --no-cpu --e2e-slabs $4 \
    > gpurun_out/${tag}_$1_$2.json 2> gpurun_out/${tag}_$1_$2.err
  grep "pipe" gpurun_out/${tag}_$1_$2.err | tail -60 > gpurun_out/${tag}_$1_$2_pipe.txt
done
echo done
