# N-rank bench path on ONE GPU (gloo for the harness collectives, both ranks on device 0):
# validates the torchrun launch, the mailbox connection and the JSON line (timings are not meaningful).
cd $GRAFT_REPO_ROOT
export FCM_BENCH_DIST_BACKEND=gloo FCM_BENCH_DEVICE_MODULO=1
for tr in p2p; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
   bench.py --gpus 2 --config C2 --steps 5 --warmup 3 --transport $tr > gpurun_out/b2_$tr.json 2> gpurun_out/b2_$tr.err
echo "rc=$?"; cat gpurun_out/b2_$tr.json | cut -c1-600; tail -3 gpurun_out/b2_$tr.err
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 \
   bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/b2_ref.json 2> gpurun_out/b2_ref.err
echo "ref rc=$?"; cut -c1-300 gpurun_out/b2_ref.json
