# one short bench line per BASELINE config (throughput context for the non-headline rows)
for wl in ${WL:-C1 C2 C3 C5}; do
  echo "$wl $(timeout 600 python bench.py --workload $wl --steps ${STEPS:-3} --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value'],3), round(d['ms_per_step'],2), r['busy_share_of_step'], r['kernel'], round(r['avg_launch_ms']*1e3,1), 'frac', round(r['frac'],3), 'step', round(r['step']['frac'],3), 'work', round(r['work_fraction'],3))")"
done
