# A/B of programmatic dependent launch (PCB_PDL) on the bench step; extra env via $1
cd $GRAFT_REPO_ROOT
for v in 0 1 0 1; do echo "$1 PCB_PDL=$v"; env $1 PCB_PDL=$v python bench.py --steps 40 --warmup 5 --no-cpu --no-e2e --no-ttc ${2:-} | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][0]); print(d['ms_per_step'], d['roofline']['per_family_ms'])"; done
