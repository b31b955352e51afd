mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "topk or deviation_topk or attention" 2>&1 | tail -5
bash tools/gpu/sanitize.sh
for shp in "553 4096 4096 1 1" "553 6144 4096 1 0" "553 4096 14336 1 1"; do
  echo "== trace $shp"; python tools/gemm_trace.py $shp 2>&1 | head -80
done > gpurun_out/r02c_gemm_traces.txt
