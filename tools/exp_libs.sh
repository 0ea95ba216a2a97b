# timing experiments: swap in variant libraries (built with -DCOFEM_TC_EXP_*; results numerically invalid)
cp paper_2202_12808_b200/libcofem.so /tmp/libcofem_ref.so
for v in ${VARIANTS}; do
  cp tools/libcofem_$v.so paper_2202_12808_b200/libcofem.so; touch paper_2202_12808_b200/libcofem.so
  echo "$v $(WL=${WL:-C3} STEPS=1 bash tools/bench_all.sh)"
done
cp /tmp/libcofem_ref.so paper_2202_12808_b200/libcofem.so; touch paper_2202_12808_b200/libcofem.so
