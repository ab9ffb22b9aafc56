for i in 1 2 3 4 5 6; do timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "longnet_block_partials" 2>&1 | tail -1; done
echo CPASYNC
for i in 1 2 3; do GA_LNET_CPASYNC=1 timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "longnet_block_partials" 2>&1 | tail -1; done
echo FULLFILE
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "longnet" 2>&1 | tail -2
