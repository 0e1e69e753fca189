timeout 600 python -m pytest tests/test_gpu_sharding.py -q -x 2>&1 | tail -3
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-forward --soak-s 0.2 2>&1 | grep '^{' | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['value'], d['ms_per_step'], d['scaling'], d['sharding'], d['roofline']['frac'], d['e2e']['value'])"
ATMM_BENCH_DIST=gloo timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 50 --warmup 5 --no-forward --soak-s 0.2 2>&1 | grep '^{' | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('N2 gloo', d['value'], d['ms_per_step'], d['scaling'], d['sharding'], d['n_gpus'])"
ATMM_BENCH_DIST=gloo timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --strong --config cfg5 --steps 20 --warmup 3 --no-forward --soak-s 0.2 2>&1 | grep '^{' | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('N2 strong cfg5', d['value'], d['ms_per_step'], d['scaling'], d['sharding'])"
