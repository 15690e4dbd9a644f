# Build a variant of libclomp_b200.so with extra -D flags on one source file
# (experiment driver): tools/variant.sh NAME SOURCE.cu "-DFOO=1 ..."
# -> variants/NAME.so (the other objects come from the current _build/).
set -e
name=$1; src=$2; flags=$3
R=$(cd "$(dirname "$0")/.." && pwd)
B=$R/paper_2501_11592_b200/_build
mkdir -p $R/variants /tmp/variants/$name
stem=$(basename $src .cu)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  --expt-relaxed-constexpr -I$R/include -I$R/paper_2501_11592_b200/csrc $flags \
  -c $R/paper_2501_11592_b200/csrc/$src -o /tmp/variants/$name/$stem.o
objs=""
for o in $B/*.o; do
  if [ "$(basename $o)" = "$stem.o" ]; then objs="$objs /tmp/variants/$name/$stem.o"; else objs="$objs $o"; fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $R/variants/$name.so $objs -lpthread -ldl -lrt
echo built variants/$name.so
