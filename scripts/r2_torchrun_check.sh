# r2_torchrun_check.sh : the driver's multi-rank launch line with one rank (contract check of both arms)
mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/torchrun_bench.json 2> gpurun_out/torchrun_bench.err; echo rc=$?
python -c "import json; d=json.loads(open('gpurun_out/torchrun_bench.json').read().strip().splitlines()[-1]); print({k: d[k] for k in ('metric','value','n_gpus','steps','warmup','scaling','gpu_launches')}, d['e2e']['value'], d['roofline']['frac'], d['cpu_baseline']['value'])"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > gpurun_out/torchrun_ref.json 2> gpurun_out/torchrun_ref.err; echo rc=$?
tail -c 300 gpurun_out/torchrun_ref.json
