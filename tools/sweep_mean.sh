# tuning sweep: SMs given to the concurrent fp64 mean column of the 1024-DCT path (0 = all)
for v in ${MS:-0 18 37 74}; do
  echo "mean_sms=$v $(COFEM_1K_MEAN_SMS=$v python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value'],2), round(d['ms_per_step'],2), r['share_of_step'])")"
done
