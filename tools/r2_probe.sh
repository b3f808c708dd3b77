# round-2 probe batch (run on the GPU box through gpurun)
set -u
mkdir -p gpurun_out
timeout 300 ./build_variants/gather_probe > gpurun_out/r2_gather.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_solver_parity.py -x -q -m gpu -rs --durations=10 -k "512 or bicgstab" > gpurun_out/r2_solver_parity2.log 2>&1
timeout 300 python bench.py --quick --steps 10 --warmup 3 > gpurun_out/r2_bq.json 2> gpurun_out/r2_bq.err
WK_DIST_BACKEND=gloo timeout 600 python bench.py --gpus 2 --steps 4 --warmup 3 > gpurun_out/r2_b2.json 2> gpurun_out/r2_b2.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r2_bref.json 2> gpurun_out/r2_bref.err
