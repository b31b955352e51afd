mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q 2>&1 | tail -4
for shp in "553 4096 4096 1 1" "553 6144 4096 1 0" "553 4096 14336 1 1"; do
  echo "== trace $shp"; python tools/gemm_trace.py $shp 2>&1 | head -10
done > gpurun_out/r02h_gemm_traces.txt
head -36 gpurun_out/r02h_gemm_traces.txt
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02h_bench.json 2> gpurun_out/r02h_bench.err
python -c "import json;d=json.loads(open('gpurun_out/r02h_bench.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['value'],d['kernel_ms'],d['roofline']['frac'],d['roofline']['path']['frac'])"
