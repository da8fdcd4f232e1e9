timeout 900 python -m pytest -q -x tests/test_conv_f32.py tests/test_dropin_cpp.py 2>&1 | grep -E "Error|error|assert|FAILED|passed|failed" | head -20
./tests/cpp/_build/dropin_parity | grep -E "fast conv|DROPIN"
