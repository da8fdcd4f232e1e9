# Round-2 compute-sanitizer sweep: memcheck over the split-precision (x2) kernels and the fp32 net,
# racecheck (shared-memory hazards) and synccheck (barrier misuse) over the fused tcgen05 kernels,
# the reference-layout operators and the net layers, at small sizes. Summary: gpurun_out/sanitizer_r2.txt
mkdir -p gpurun_out
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
out=gpurun_out/sanitizer_r2.txt; : > $out
run() {  # tool, name, pytest args...
  tool=$1; name=$2; shift 2
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 \
    python -m pytest -q -x -p no:cacheprovider "$@" > gpurun_out/san_${tool}_$name.log 2>&1
  echo "$tool $name rc=$? $(grep -E 'passed|failed' gpurun_out/san_${tool}_$name.log | tail -1) | $(grep 'ERROR SUMMARY' gpurun_out/san_${tool}_$name.log | tail -1)" >> $out
}
run memcheck conv_f32 tests/test_conv_f32.py -k "random_maps or tiny_and_ragged or empty_and_errors or split_planes"
run memcheck net_f32 tests/test_net_gpu.py -k "f32"
run racecheck conv_tc tests/test_conv_tc.py -k "tiny_and_ragged or random_maps"
run racecheck conv_f32 tests/test_conv_f32.py -k "random_maps or tiny_and_ragged"
run racecheck ops_ref tests/test_ops_gpu.py -k "golden_instance_bit_exact or kat"
run racecheck net tests/test_net_gpu.py -k "pool_unpool or bn_relu"
run synccheck conv_tc tests/test_conv_tc.py -k "tiny_and_ragged or random_maps"
run synccheck conv_f32 tests/test_conv_f32.py -k "random_maps or tiny_and_ragged"
run synccheck ops_ref tests/test_ops_gpu.py -k "golden_instance_bit_exact or kat"
run synccheck net tests/test_net_gpu.py -k "pool_unpool or bn_relu"
cat $out
