timeout 150 python tools/wtc_tiny.py 2048 1 > /dev/null || { echo "tiny case failed/hung"; exit 1; }
timeout 900 python -m pytest tests/test_gpu_edgesets.py tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_contracts.py tests/test_gpu_variants.py -q -x -p no:cacheprovider -k "csr or CSR or coo or COO or heavy" 2>&1 | tail -n 2
