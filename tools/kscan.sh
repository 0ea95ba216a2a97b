for K in 4 8 16 32; do
 for l in tools/libcofem_noflow.so tools/libcofem_v3.so; do
  cp $l paper_2202_12808_b200/libcofem.so
  echo "K=$K $l $(TIME_K=$K timeout 60 python tools/time_estep.py C4 3 /tmp/a_C4.pt 2>&1 | tail -1 | sed 's/.*median//; s/frozen.*//')"
 done
done
