bash tools/gpu_variants.sh a3 "base arena" "C1 dilate 3" "C1 erode 3" "C2 dilate 4" "C2 shell 4" "C3 dilate 8" "C4 dilate 1" "C4 dilate 16" "C5 shell 16"
cp exp/libdexel_arena.so paper_1804_08968_b200/libdexel.so; touch paper_1804_08968_b200/libdexel.so
DEXEL_DEBUG=1 timeout 300 python tools/time_op.py C1 dilate 3 3 > gpurun_out/a3_arena_debug_c1.log 2>&1
DEXEL_DEBUG=1 timeout 300 python tools/time_op.py C2 shell 4 3 > gpurun_out/a3_arena_debug_c2.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/a3_arena_pytest_full.log 2>&1; echo "pytest rc=$?" >> gpurun_out/a3_arena_pytest_full.log
