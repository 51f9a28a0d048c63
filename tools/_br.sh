bash tools/gpu_tests.sh br
for i in 1 2; do
timeout 600 python tools/c5_timed.py 300 20 2>&1 | tail -1 | cut -c1-130
DSMC_NO_BRANCH=1 timeout 600 python tools/c5_timed.py 300 20 2>&1 | tail -1 | cut -c1-130
done
for c in c2; do timeout 600 python bench.py --config c2 --steps 20 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | cut -c100-260; DSMC_NO_BRANCH=1 timeout 600 python bench.py --config c2 --steps 20 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | cut -c100-260; done
