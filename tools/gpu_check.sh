mkdir -p gpurun_out
for w in 3 8 3 8; do FC_GRAM_WAVES=$w timeout 120 python bench.py --steps 5 --warmup 3 2>>gpurun_out/bench.err | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('w$w', d['value'], d['ms_per_step'], d['final_rel_res'])" || exit 1; done
