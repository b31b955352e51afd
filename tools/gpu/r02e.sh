mkdir -p gpurun_out
python tools/topk_debug.py 2>&1 | tail -12
for shp in "553 4096 4096 1 1" "553 6144 4096 1 0" "553 4096 14336 1 1"; do
  echo "== trace $shp"; python tools/gemm_trace.py $shp 2>&1 | head -12
done > gpurun_out/r02e_gemm_traces.txt
head -40 gpurun_out/r02e_gemm_traces.txt
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02e_bench.json 2> gpurun_out/r02e_bench.err
tail -c 2500 gpurun_out/r02e_bench.json
