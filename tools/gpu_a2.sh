timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "rasterize" > gpurun_out/a2_pytest_raster.log 2>&1; echo "pytest rc=$?" >> gpurun_out/a2_pytest_raster.log
python bench.py --config C3 --op rasterize --steps 5 --warmup 3 > gpurun_out/a2_bench_c3_raster.json 2> gpurun_out/a2_bench_c3_raster.err
bash tools/gpu_variants.sh a2 "base pre" "C5 shell 16" "C4 dilate 16" "C4 dilate 64" "C3 dilate 8" "C2 shell 4"
