# e2e (pinned host -> pinned host gridrec) per host-pipeline chunk schedule
run() { SPTB_PIPE_SIZES="$1" timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-solvers --no-parity --pipeline-slices 0 > gpurun_out/e2e_s.json 2>/dev/null; python -c "import json;d=json.loads(open('gpurun_out/e2e_s.json').read().strip().splitlines()[-1]);e=d['e2e'];print('$1', round(e['ms_per_step'],3), round(e['value']), round(e['pcie_roofline']['duplex_ms'],3), round(e['frac_of_pcie_bound'],4))"; }
run "1"
run "1,4,4,4,4,4,4,4,2,1"
run "1,2,2,2,2,2,2,2,2,2,2,2,2,2,2,2,1"
run "1,1,2,4,4,4,4,4,4,2,1,1"
run "1,1,2,2,2,2,2,2,2,2,2,2,2,2,2,1,1,1"
run "1"
