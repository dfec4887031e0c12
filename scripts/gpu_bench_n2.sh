# N > 1 bench path on one GPU (ENERGON_BENCH_SHARE_GPU=1: both ranks on cuda:0, gloo plumbing, P2P exchange)
ENERGON_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 --layers 4 > gpurun_out/bench_n2.log 2>&1; echo "rc=$?"; tail -c 1500 gpurun_out/bench_n2.log
