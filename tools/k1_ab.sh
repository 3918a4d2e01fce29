timeout 600 python -m pytest tests -m gpu -x -q --timeout 300 -p no:cacheprovider -k "parity or ingest or extremes" > gpurun_out/k1_pytest.log 2>&1; tail -2 gpurun_out/k1_pytest.log
VARS="${VARS:-old u4 u8m2 u16m2}" bash tools/abl_k2.sh
