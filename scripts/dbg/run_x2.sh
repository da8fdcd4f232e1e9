timeout 600 python -m pytest -q tests/test_ops_gpu.py -k "stream_ordered or errors_mirror" 2>&1 | tail -2
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/b1.json; python -c "
import json; d=json.load(open('gpurun_out/b1.json')); print(d['ms_per_step'], d['e2e']['ms_per_step'], json.dumps(d['ref_layout_kernels'])[:900]); print(d['roofline'])"
HCB_TEST_SHARE_GPU=1 HCB_TEST_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --res 64 --no-cpu-baseline --no-ref-kernels 2>&1 | tail -3 | cut -c1-400
