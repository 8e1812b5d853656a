set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r01f.log 2>&1; tail -3 gpurun_out/pytest_gpu_r01f.log
timeout 900 python bench.py > gpurun_out/bench_r01f.json 2> gpurun_out/bench_r01f.err; tail -3 gpurun_out/bench_r01f.err
timeout 1200 bash tools/profile_round.sh r01f
