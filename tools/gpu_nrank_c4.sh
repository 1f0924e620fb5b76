# N-rank bench path at C4 (large volume: owner path, in-loop seeded start) with both ranks on ONE GPU
# (gloo for the harness collectives): validates the multi-rank fused exchange end to end at the headline
# size (timings are not meaningful: the two cooperative kernels share the GPU).
cd $GRAFT_REPO_ROOT
export FCM_BENCH_DIST_BACKEND=gloo FCM_BENCH_DEVICE_MODULO=1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 \
   bench.py --gpus 2 --config C4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/b2_c4.json 2> gpurun_out/b2_c4.err
echo "rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/b2_c4.json')); print({k: d.get(k) for k in ('value','ms_per_step','n_gpus','gpu_launches')}, d['config'].get('iterations_per_solve'))"; tail -3 gpurun_out/b2_c4.err
