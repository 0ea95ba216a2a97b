# timing-experiment builds of the dense tcgen05 path (numerically INVALID): each variant
# disables one pipeline component with -DCOFEM_TC_EXP_<V> (V1+V2 combines); the library goes to tools/libcofem_<v>.so
set -e
cd "$(dirname "$0")/.."
python -c "from paper_2202_12808_b200 import build; build.build()"
B=paper_2202_12808_b200/_build
for v in ${VARIANTS:-NOTMA NOPROMO TRACE}; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    -I include $(echo $v | sed 's/^/-DCOFEM_TC_EXP_/; s/+/ -DCOFEM_TC_EXP_/g') -c paper_2202_12808_b200/csrc/op_dense_tc.cu -o /tmp/tc_$v.o
  objs=$(ls $B/*.o | grep -v op_dense_tc.o)
  /usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a -o tools/libcofem_$v.so $objs /tmp/tc_$v.o -lcudart
done
