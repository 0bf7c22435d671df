set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
nproc; free -g | head -2
timeout 1200 python -m pytest tests -q -m gpu -p pytest_timeout --timeout 600 -x 2>&1 | tail -40 > gpurun_out/pytest_gpu.txt; cat gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 600 python bench.py --slits 8 --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -5 | tee gpurun_out/bench_small.txt
