# GPU round script (gpurun): tests, then the headline bench, then the launch profile
set -x
mkdir -p gpurun_out
TAG=${TAG:-r2}
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/${TAG}_gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${TAG}_gputests.log
tail -15 gpurun_out/${TAG}_gputests.log
for c in ${CONFIGS:-cfg5bt}; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
  python -c "import json;d=json.load(open('gpurun_out/${TAG}_bench_$c.json'));print('$c', d['ms_per_step'], d['e2e']['value'], d['amplitude'])"
  timeout 300 python tools/launch_profile.py --config $c > gpurun_out/${TAG}_launch_profile_$c.txt 2>&1
  head -30 gpurun_out/${TAG}_launch_profile_$c.txt
done
