# Timing-experiment build: recompile one source of the library with extra -D flags and link
# tools/libcofem_<name>.so from the in-tree objects (used with tools/ab_time.sh).
#   bash tools/build_variant.sh op_dct1k.cu PFD2 -DCOFEM_1K_PFD=2
set -e
cd "$(dirname "$0")/.."
src=$1; name=$2; shift 2
python -c "from paper_2202_12808_b200 import build; build.build()" > /dev/null
B=paper_2202_12808_b200/_build
base=$(basename $src .cu)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -I include "$@" -c paper_2202_12808_b200/csrc/$src -o /tmp/var_$name.o
objs=$(ls $B/*.o | grep -v "/$base.o")
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a -o tools/libcofem_$name.so $objs /tmp/var_$name.o -lcudart
echo tools/libcofem_$name.so
