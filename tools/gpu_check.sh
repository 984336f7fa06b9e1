mkdir -p gpurun_out
python bench.py --steps 3 --warmup 3 > gpurun_out/bench.jsonl 2> gpurun_out/bench.err
tail -1 gpurun_out/bench.jsonl
