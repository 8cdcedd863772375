for c in c1 c2; do
python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-lifted > gpurun_out/b.json 2> gpurun_out/b.err; python -c "import json; d=json.load(open('gpurun_out/b.json')); print('$c graph', d['value'], d['phases_ms'])"
CKKT_NO_GRAPH=1 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-lifted > gpurun_out/b.json 2> gpurun_out/b.err; python -c "import json; d=json.load(open('gpurun_out/b.json')); print('$c nograph', d['value'], d['phases_ms'])"
done
