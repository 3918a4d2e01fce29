timeout 600 python -m pytest tests -m gpu -x -q --timeout 300 -p no:cacheprovider -k "filter or parity or shard" > gpurun_out/f_pytest.log 2>&1; tail -2 gpurun_out/f_pytest.log
VARS="${VARS:-p0 p1 p3 p4}" bash tools/abl_k2.sh
for d in uniform_disk gaussian; do echo -n "$d "; DIST=$d timeout 300 python tools/knob_sweep.py X=0; done
