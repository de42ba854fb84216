# A/B timing of kernel_cluster.cu build variants: each variant is a comma-separated list
# of macro assignments (DVW_DIAG=<mask> diagnostic builds -- wrong codes, timing only; DVW_EXP,
# DVW_CHAIN0, DVW_DEADFLAG, DVW_SKIPSTAGE switches); "base" = the in-tree defaults.  Rebuilds only
# kernel_cluster.cu into scratch copies of the package and times C2 / C3 with each.
#   bash tools/diag_c2.sh "base DVW_DIAG=16 DVW_CHAIN0=0,DVW_EXP=2" gpurun_out/diag   (build first)
set -e
VARS=${1:-"base"}
OUT=${2:-gpurun_out/diag}
NV=/usr/local/cuda/bin/nvcc
mkdir -p $OUT
i=0
for V in $VARS; do
  i=$((i+1))
  D=/tmp/dvw_diag_$i
  rm -rf $D; mkdir -p $D
  cp -r paper_1702_07825_b200 include $D/
  C=$D/paper_1702_07825_b200/csrc
  DEFS=""
  if [ "$V" != "base" ]; then DEFS=$(echo $V | tr ',' '\n' | sed 's/^/-D/' | tr '\n' ' '); fi
  $NV -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-fvisibility=hidden \
      --expt-relaxed-constexpr -I $D/include $DEFS -c $C/kernel_cluster.cu -o $C/kernel_cluster.o
  $NV -gencode arch=compute_100a,code=sm_100a -shared -o $D/paper_1702_07825_b200/libdvw.so $C/*.o -lcuda
  echo "== $V" >> $OUT/diag.txt
  if [ -n "$DIAG_CMD" ]; then
    (cd $D && cp -r /root/repo/bench.py /root/repo/oracle . 2>/dev/null; DVW_PKG_ROOT=$D timeout 600 bash -c "$DIAG_CMD") >> $OUT/diag.txt 2>&1
  else
    DVW_PKG_ROOT=$D timeout 300 python tools/sweep_layers.py --layers ${LAYERS:-20,40} --n 8000 >> $OUT/diag.txt 2>&1
  fi
done
cat $OUT/diag.txt
