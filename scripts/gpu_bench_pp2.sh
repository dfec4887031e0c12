# NBPP bench path on one GPU (ENERGON_BENCH_SHARE_GPU=1): 2 stages in 2 processes sharing cuda:0
ENERGON_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --pp 2 --pp-batches 6 --warmup 2 --layers 4 > gpurun_out/bench_pp2.log 2>&1; echo "rc=$?"; tail -c 1800 gpurun_out/bench_pp2.log
