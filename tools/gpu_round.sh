set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2_gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2_gputests.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench_cfg5bt.json 2> gpurun_out/r2_bench_cfg5bt.err
python tools/launch_profile.py --config cfg5bt > gpurun_out/r2_launch_profile_cfg5bt.txt 2>&1
tail -3 gpurun_out/r2_gputests.log; cat gpurun_out/r2_bench_cfg5bt.json | head -c 3000
