# compute-sanitizer memcheck over the GPU parity tests at small sizes (run under gpurun);
# summary lines go to gpurun_out/sanitizer.txt
mkdir -p gpurun_out
export PYTORCH_NO_CUDA_MEMORY_CACHING=1  # exact cudaMalloc per tensor, so overruns are visible to memcheck
out=gpurun_out/sanitizer.txt; : > $out
run() {  # name, pytest args...
  name=$1; shift
  timeout 1200 compute-sanitizer --tool memcheck --leak-check no --print-limit 20 --error-exitcode 9 \
    python -m pytest -q -x -p no:cacheprovider "$@" > gpurun_out/san_$name.log 2>&1
  echo "$name rc=$? $(grep -E 'passed|failed' gpurun_out/san_$name.log | tail -1) | $(grep 'ERROR SUMMARY' gpurun_out/san_$name.log | tail -1)" >> $out
}
run conv_tc tests/test_conv_tc.py -k "tiny_and_ragged or empty_batch or deconv or random_maps or argument_errors"
run gemm_tc tests/test_gemm_tc.py -k "7-36-132 or 5-33-77 or 8-2000-100 or 64-300-132 or 9-40-1001 or truncates or 16-216-3680"
run ops_ref tests/test_ops_gpu.py -k "golden_instance_bit_exact or random_batches or kat"
run ops_f64 tests/test_ops_f64_gpu.py
run net tests/test_net_gpu.py -k "pool_unpool or bn_relu or descends"
run psh tests/test_psh_device.py -k "16-300 or 32-3000"
cat $out
