# bench modes: default N=1, Ulysses at N=1 (chunked pipeline, P=1), and 2-rank gloo bring-up runs on one GPU
mkdir -p gpurun_out
python -m paper_2601_11641_b200.build > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
show() { grep "^{" $1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print('$2', 'n', d['n_gpus'], 'value', d['value'], 'ms', d['ms_per_step'], 'attn_ms', d['attn_ms'], 'frac', d['roofline']['frac'], 'e2e', d['e2e'] and d['e2e']['ms_per_step'], d['config'].get('parallelism'), d['config'].get('lpt'), 'traffic', d['roofline']['traffic'])" || tail -5 $1; }
timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bm_default.log 2>&1; show gpurun_out/bm_default.log default
timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu --no-dense --ulysses > gpurun_out/bm_uly1.log 2>&1; show gpurun_out/bm_uly1.log ulysses1
MOD_BENCH_DIST_BACKEND=gloo timeout 600 python bench.py --gpus 2 --steps 2 --warmup 3 --no-cpu --no-dense --no-e2e --config cogvideox-5b --lpt > gpurun_out/bm_lpt2.log 2>&1; show gpurun_out/bm_lpt2.log lpt2_gloo
MOD_BENCH_DIST_BACKEND=gloo timeout 600 python bench.py --gpus 2 --steps 2 --warmup 3 --no-cpu --no-dense --config cogvideox-5b --ulysses > gpurun_out/bm_uly2.log 2>&1; show gpurun_out/bm_uly2.log uly2_gloo
