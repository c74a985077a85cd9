# multi-rank code path of bench.py on a 1-GPU box: N ranks share the GPU, gloo for the scalar
# reductions (MOD_BENCH_DIST_BACKEND=gloo).  Validates the N>1 logic only; the numbers are meaningless.
mkdir -p gpurun_out
for n in 2 4; do
MOD_BENCH_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2951$n bench.py --gpus $n --steps 3 --warmup 3 --no-dense > gpurun_out/multirank_$n.log 2>&1; echo "n=$n rc=$?"
grep '^{' gpurun_out/multirank_$n.log | cut -c1-600; grep -i "error\|Traceback" gpurun_out/multirank_$n.log | head -5
MOD_BENCH_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2952$n bench.py --impl reference --gpus $n --steps 2 --warmup 1 > gpurun_out/multirank_ref_$n.log 2>&1; echo "ref n=$n rc=$?"; grep '^{' gpurun_out/multirank_ref_$n.log | cut -c1-300
done
