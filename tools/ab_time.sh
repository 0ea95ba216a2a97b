# A/B timing of library variants on one box: for each .so in $LIBS (paths), install it as the
# in-tree libcofem.so and time a fixed-alpha E-step of $WL (tools/time_estep.py), twice, interleaved.
WL=${WL:-C4}
cp paper_2202_12808_b200/libcofem.so /tmp/libcofem_orig.so
python tools/time_estep.py $WL 3 /tmp/a_$WL.pt > /dev/null 2>&1
for rep in 1 2; do
  for l in $LIBS; do
    cp $l paper_2202_12808_b200/libcofem.so
    echo "$l: $(python tools/time_estep.py $WL ${REPS:-5} /tmp/a_$WL.pt 2>&1 | tail -1)"
  done
done
cp /tmp/libcofem_orig.so paper_2202_12808_b200/libcofem.so
