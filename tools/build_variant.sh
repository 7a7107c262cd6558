#!/bin/bash
# build_variant.sh NAME [nvcc -D flags...] -> paper_1406_5687_b200/variants/lib_NAME.so (dev experiments)
set -e
cd "$(dirname "$0")/../paper_1406_5687_b200"
name=$1; shift
tmp=/tmp/vb_$name; rm -rf $tmp; mkdir -p $tmp variants
for f in csrc/*.cu; do
  b=$(basename $f .cu)
  /usr/local/cuda/bin/nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-O3 \
    --expt-relaxed-constexpr -Xptxas -v -I../include "$@" -c $f -o $tmp/$b.o 2>$tmp/$b.log &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/lib_$name.so $tmp/*.o -lcudart_static -lrt -lpthread -ldl
echo "$name: $(grep -E -A3 'k_(engine|small)INS_8PullSegs' $tmp/count.log | grep -E 'Used|spill' | tr -s ' ' | tr '\n' ' ')"
