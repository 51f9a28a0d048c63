# usage: bash tools/gpu_contract.sh -- the driver's bench invocations (reference arm, torchrun N=1, smoke)
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 2>&1 | tail -1 | cut -c1-300
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu 2>&1 | grep '^{' | cut -c1-300
