set -x
python -m pytest tests/test_gpu_decisions.py -q -x 2>&1 | tail -2
python tools/score_bench.py 2>&1 | tail -1 | cut -c1-200
timeout 180 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 tools/c4_peer.py 300 --gpus 1024 --one-gpu --check 2>&1 | grep -v Warning | tail -5
nvidia-smi --query-gpu=name,utilization.gpu --format=csv
