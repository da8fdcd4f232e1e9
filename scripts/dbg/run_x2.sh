timeout 600 python -m pytest -q tests/test_dp_host.py 2>&1 | tail -3
RANK=0 WORLD_SIZE=1 LOCAL_RANK=0 timeout 300 ./hosts/_build/dp_conv --psh paper_1803_11385_b200/_cache/shell256_l01.psh --steps 20 --warmup 5
