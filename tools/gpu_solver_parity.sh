nproc > gpurun_out/r2_box.txt; free -g >> gpurun_out/r2_box.txt; lscpu | head -20 >> gpurun_out/r2_box.txt; nvidia-smi >> gpurun_out/r2_box.txt
timeout 1500 python -m pytest tests/test_gpu_solver_parity.py -x -q -m gpu -rs --durations=10 > gpurun_out/r2_solver_parity.log 2>&1
echo rc=$? >> gpurun_out/r2_solver_parity.log
