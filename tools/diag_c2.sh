# Timing diagnostics of the batch-1 cluster kernel: rebuild kernel_cluster.cu with
# -DDVW_DIAG=<mask> into scratch copies of the package and time C2 / C3 with each.  Codes are wrong
# in the diagnostic builds; only the timing means anything.
#   bash tools/diag_c2.sh "0 1 2 4 8 16" gpurun_out/diag      (needs the in-tree .o files: build first)
set -e
MASKS=${1:-"0 1 2 4 8 16"}
OUT=${2:-gpurun_out/diag}
NV=/usr/local/cuda/bin/nvcc
mkdir -p $OUT
for M in $MASKS; do
  D=/tmp/dvw_diag_$M
  rm -rf $D; mkdir -p $D
  cp -r paper_1702_07825_b200 include $D/
  C=$D/paper_1702_07825_b200/csrc
  $NV -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-fvisibility=hidden \
      --expt-relaxed-constexpr -I $D/include -DDVW_DIAG=$M -c $C/kernel_cluster.cu -o $C/kernel_cluster.o
  $NV -gencode arch=compute_100a,code=sm_100a -shared -o $D/paper_1702_07825_b200/libdvw.so $C/*.o -lcuda
  touch $D/paper_1702_07825_b200/libdvw.so
  echo "== DVW_DIAG=$M" >> $OUT/diag.txt
  DVW_PKG_ROOT=$D timeout 300 python tools/sweep_layers.py --layers 20,40 --n 8000 >> $OUT/diag.txt 2>&1
done
cat $OUT/diag.txt
