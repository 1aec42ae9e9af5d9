mkdir -p gpurun_out
for m in 512 4096; do timeout 1200 python tools/dense_error.py --m $m --rows 200000; done > gpurun_out/dense_error.jsonl 2> gpurun_out/dense_error.err
cat gpurun_out/dense_error.jsonl; tail -3 gpurun_out/dense_error.err
