set -x
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q tests/test_conv_f32.py tests/test_dropin_cpp.py tests/test_ops_gpu.py 2>&1 | tail -15
./tests/cpp/_build/dropin_parity | grep -E "fast conv|DROPIN"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 600 python bench.py --steps 20 --warmup 5 2>&1 | tail -2
timeout 600 python bench.py --steps 20 --warmup 5 --dtype bf16 --no-cpu-baseline --no-e2e 2>&1 | tail -1
