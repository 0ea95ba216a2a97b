# Round evidence refresh (run on the GPU box from the repo root): bench lines for every config,
# the ncu launch list of the headline bench, and one --set full capture per hot kernel family.
# Outputs land in gpurun_out/<tag>_*; tools/ncu_summary.py turns them into profiles/ markdown.
TAG=${TAG:-v3}
O=gpurun_out
timeout 900 python bench.py --steps 3 --warmup 3 > $O/${TAG}_bench_C4.json 2> $O/${TAG}_bench_C4.err
for wl in C1 C2 C3 C5; do
  timeout 900 python bench.py --workload $wl --steps 3 --warmup 3 --no-cpu-baseline > $O/${TAG}_bench_$wl.json 2> $O/${TAG}_bench_$wl.err
done
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > $O/${TAG}_ref_C4.json 2> $O/${TAG}_ref_C4.err
N="ncu --clock-control none"
# launch list of one E-step after the 3 warm-up ones (12 launches per CG iteration x 200 + setup)
timeout 900 $N --metrics gpu__time_duration.sum --launch-skip 7300 -c 2400 --csv --log-file $O/${TAG}_launches_C4.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-conformance > $O/${TAG}_ncu_launch.log 2>&1
# full sets of steady-state launches (--launch-skip: CG iterations with every column active; the
# first launches are iteration 0, which has no direction update)
timeout 1200 $N --set full --import-source on -k regex:"k1k_rows|k1k_cols|k_update" --launch-skip 120 -c 8 -o $O/${TAG}_C4_full \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-conformance > $O/${TAG}_ncu_c4.log 2>&1
timeout 1200 $N --set full --import-source on -k regex:"k_tc_phi|k_update|k_dir" --launch-skip 40 -c 4 -o $O/${TAG}_C3_full \
  python bench.py --workload C3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-conformance > $O/${TAG}_ncu_c3.log 2>&1
timeout 1200 $N --set full --import-source on -k regex:"k_conv_fft|k_update" --launch-skip 40 -c 4 -o $O/${TAG}_C5_full \
  python bench.py --workload C5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-conformance > $O/${TAG}_ncu_c5.log 2>&1
# afterwards, here: python tools/ncu_traffic.py C4=$O/${TAG}_C4_full.ncu-rep C3=... C5=...
ls -la $O/${TAG}_*
