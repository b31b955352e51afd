# compute-sanitizer passes over small blends (tools/sanitize_blend.py); logs -> gpurun_out/san_*.log
mkdir -p gpurun_out
python tools/sanitize_blend.py > gpurun_out/san_plain.log 2>&1; echo "plain rc=$?"
for tool in memcheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 --target-processes all \
      python tools/sanitize_blend.py > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/san_$tool.log
done
CB_SAN_NO_PDL=1 timeout 1200 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 30 \
    --target-processes all python tools/sanitize_blend.py > gpurun_out/san_racecheck.log 2>&1
echo "racecheck rc=$?"; tail -3 gpurun_out/san_racecheck.log
