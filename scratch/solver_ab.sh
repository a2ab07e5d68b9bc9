# solver iteration rates with and without an env switch (bench.py solver legs)
for v in 0 1; do
  env $1=$v timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-parity --no-e2e --pipeline-slices 0 > gpurun_out/sab_$v.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/sab_$v.json').read().strip().splitlines()[-1]);print('$1=$v', 'gridrec', round(d['ms_per_step'],3), 'sirt', round(d['sirt_iter']['ms_per_iteration'],3), 'cgls', round(d['cgls_iter']['ms_per_iteration'],3), 'tv', round(d['tv_iter']['ms_per_iteration'],3))"
done
