cd $GRAFT_REPO_ROOT
for n in 16 32 64 128; do
timeout 300 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu --no-es --no-bits --no-critical --n-seq $n > /tmp/n$n.json 2>/dev/null
python -c "import json;d=json.load(open('/tmp/n$n.json'));print($n, round(d['ms_per_step'],4), {k:round(v,4) for k,v in d['stages_ms'].items()}, d['parity']['mismatches'])"
done
