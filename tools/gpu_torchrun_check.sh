timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/torchrun_n1.log 2>&1; echo torchrun=$?
grep '^{' gpurun_out/torchrun_n1.log | tail -1 | cut -c1-600
timeout 300 python bench.py --gpus 2 --config c2 --steps 3 --warmup 3 > gpurun_out/gpus2_on_1.log 2>&1; echo gpus2=$?
tail -5 gpurun_out/gpus2_on_1.log | cut -c1-400
