# Steady-state (CG iteration >= 2) per-launch duration and DRAM bytes of the hot kernels, one
# serialised ncu pass per workload (run on the GPU box from the repo root; writes gpurun_out/).
TAG=${TAG:-steady}
O=gpurun_out
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
timeout 900 ncu --clock-control none --metrics $M -k regex:"k1k_rows|k1k_cols|k_update" --launch-skip 120 -c 24 --csv \
  --log-file $O/${TAG}_C4.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-conformance > $O/${TAG}_C4.log 2>&1
timeout 900 ncu --clock-control none --metrics $M -k regex:"k_conv_fft|k_update" --launch-skip 40 -c 12 --csv \
  --log-file $O/${TAG}_C5.csv python bench.py --workload C5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-conformance > $O/${TAG}_C5.log 2>&1
timeout 900 ncu --clock-control none --metrics $M -k regex:"k_tc_phi|k_update|k_dir" --launch-skip 40 -c 12 --csv \
  --log-file $O/${TAG}_C3.csv python bench.py --workload C3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-conformance > $O/${TAG}_C3.log 2>&1
ls -la $O/${TAG}_*
