timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu.log
WAITSIM_ENGINE=member timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_member.log 2>&1; echo pytest_member=$?
tail -2 gpurun_out/pytest_gpu_member.log
WAITSIM_ENGINE=ring timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_ring.log 2>&1; echo pytest_ring=$?
tail -2 gpurun_out/pytest_gpu_ring.log
NOTEST=1 LIBS="${LIBS:-prev cur}" WLS="${WLS:-C2 C4_2 C4_4}" bash tools/gpu_abn.sh 2>&1 | grep -v pytest | tail -40
