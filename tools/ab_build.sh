# Build kernel_cluster.cu variants LOCALLY (nvcc cross-compiles) into ab/<i>/ -- a scratch copy of
# the package + bench.py + oracle per variant -- so a gpurun call only times them (tools/ab_run.sh).
#   bash tools/ab_build.sh "base DVW_DIAG=8 DVW_DIAG=16"      (run the in-tree build first)
# Each variant is a comma-separated list of macro assignments ("base" = in-tree defaults); ab/ is
# git-ignored but travels with the gpurun snapshot.
set -e
VARS=${1:-"base"}
NV=/usr/local/cuda/bin/nvcc
rm -rf ab; mkdir -p ab
i=0
for V in $VARS; do
  i=$((i+1))
  D=ab/$i
  mkdir -p $D
  cp -r paper_1702_07825_b200 include oracle bench.py tools $D/
  rm -rf $D/tools/*.sh
  echo "$V" > $D/VARIANT
  C=$D/paper_1702_07825_b200/csrc
  DEFS=""
  if [ "$V" != "base" ]; then DEFS=$(echo $V | tr ',' '\n' | sed 's/^/-D/' | tr '\n' ' '); fi
  ( $NV -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-fvisibility=hidden \
      --expt-relaxed-constexpr -I $D/include $DEFS -c $C/kernel_cluster.cu -o $C/kernel_cluster.o && \
    $NV -gencode arch=compute_100a,code=sm_100a -shared -o $D/paper_1702_07825_b200/libdvw.so $C/*.o -lcuda && \
    touch $D/paper_1702_07825_b200/libdvw.so ) &
done
wait
ls -la ab/*/paper_1702_07825_b200/libdvw.so
