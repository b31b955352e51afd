#!/bin/bash
# after removing the off-by-default attention / top-k / GEMM experiments: GPU suite, sanitizers, bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02cr_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/r02cr_pytest_gpu.log
python tools/sanitize_blend.py > gpurun_out/r02cr_san_plain.log 2>&1; echo "plain rc=$?"
for tool in memcheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 --target-processes all \
      python tools/sanitize_blend.py > gpurun_out/r02cr_san_$tool.log 2>&1
  echo "$tool rc=$?"; tail -2 gpurun_out/r02cr_san_$tool.log
done
CB_SAN_NO_PDL=1 timeout 1200 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 30 \
    --target-processes all python tools/sanitize_blend.py > gpurun_out/r02cr_san_racecheck.log 2>&1
echo "racecheck rc=$?"; tail -2 gpurun_out/r02cr_san_racecheck.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02cr_bench.json 2> gpurun_out/r02cr_bench.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r02cr_bench.json').read().strip().splitlines()[-1]);print('mistral', d['ms_per_step'], d['value'], d['roofline']['frac'], d['roofline']['attention']['frac'], d['e2e']['ms'], d['e2e'].get('paired_overhead_ms'), d['clocks'])"
