# tuning sweep: CTA slots per SM of the persistent 1024-DCT kernels (0 = one CTA per work item),
# and the mean column serialised on the main stream (COFEM_1K_SERIAL)
for v in ${SLOTS:-0 4}; do
  for ser in ${SERIAL:-0}; do
    if [ "$ser" = 1 ]; then export COFEM_1K_SERIAL=1; else unset COFEM_1K_SERIAL; fi
    echo "slots=$v serial=$ser $(COFEM_1K_SLOTS=$v python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value'],2), round(d['ms_per_step'],2), r['share_of_step'], r['kernel'], round(r['avg_launch_ms']*1e3,1), round(r['frac'],3))")"
  done
done
