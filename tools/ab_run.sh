# Time every variant built by tools/ab_build.sh with the command in $AB_CMD (run from the variant's
# directory), appending to $1 (default gpurun_out/ab/ab.txt).
OUT=${1:-gpurun_out/ab/ab.txt}
mkdir -p $(dirname $OUT)
for D in ab/*/; do
  echo "== $(cat $D/VARIANT)" >> $OUT
  (cd $D && timeout ${AB_TIMEOUT:-600} bash -c "$AB_CMD") >> $OUT 2>&1
done
cat $OUT
