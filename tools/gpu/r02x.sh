mkdir -p gpurun_out
timeout 900 python bench.py --attn-deviation --config small > gpurun_out/r02x_attn_dev_small.json 2> gpurun_out/r02x_attn_dev_small.err; tail -3 gpurun_out/r02x_attn_dev_small.err; cat gpurun_out/r02x_attn_dev_small.json
timeout 1200 python bench.py --attn-deviation --config mistral > gpurun_out/r02x_attn_dev_mistral.json 2> gpurun_out/r02x_attn_dev_mistral.err; tail -3 gpurun_out/r02x_attn_dev_mistral.err; cat gpurun_out/r02x_attn_dev_mistral.json
