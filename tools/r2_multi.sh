python -c "import __graft_entry__ as g; g.build()" > /dev/null
export GA_DIST_BACKEND=gloo GA_FORCE_DEVICE=0
for args in "--config cfg4" "--config cfg2" "--config cfg5 --scaling strong" "--config cfg3"; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --no-e2e $args > gpurun_out/multi.json 2> gpurun_out/multi.err
echo "== $args rc=$?"; tail -c 300 gpurun_out/multi.err | tail -2
python -c "
import json; d=json.loads(open('gpurun_out/multi.json').read().strip().splitlines()[-1])
print(d['n_gpus'], d['scaling'], d['config']['workload'], round(d['ms_per_step'],3), '%.3e'%d['value'])"
done
