timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu.log
WAITSIM_ENGINE=member timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_member.log 2>&1; echo pytest_member=$?
tail -3 gpurun_out/pytest_gpu_member.log
LIBS="prev cur" WLS="${WLS:-C2 C4_2 C4_4}" bash tools/gpu_abn.sh 2>&1 | grep -v pytest | tail -20
