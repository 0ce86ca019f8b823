mkdir -p gpurun_out
python bench.py > gpurun_out/s2_bench2.json 2> gpurun_out/s2_bench2.err
python - <<'PY'
import json
d=json.load(open('gpurun_out/s2_bench2.json'))
print(d['value'], d['e2e']['value'], json.dumps(d['e2e']['pcie']))
PY
for n in 2 4 8; do
python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2950$n bench.py --gpus $n --steps 10 --warmup 3 --share-gpu > gpurun_out/s2_share_gpu_$n.json 2> gpurun_out/s2_share_gpu_$n.err
tail -c 600 gpurun_out/s2_share_gpu_$n.err
python - <<PY
import json
d=json.load(open('gpurun_out/s2_share_gpu_$n.json'))
print($n, d['value'], d['ms_per_step'], d['gpu_launches'], d['digest_checksum'], d['e2e']['value'])
PY
done
