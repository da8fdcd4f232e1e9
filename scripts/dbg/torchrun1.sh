# the driver's N>1 launch form at N=1 (NCCL process group, max-over-ranks timing path)
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/tr1.json 2> gpurun_out/tr1.err; echo "torchrun bench rc=$?"; tail -c 600 gpurun_out/tr1.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > gpurun_out/tr1_ref.json 2> gpurun_out/tr1_ref.err; echo "torchrun ref rc=$?"; tail -c 300 gpurun_out/tr1_ref.json
grep -i "nccl\|world" gpurun_out/tr1.err | head -5
