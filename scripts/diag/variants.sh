# Diag helper: run a command once per variant library (paper_2605_10501_b200/_lib/diag/lib_<V>.so).
# Usage: variants.sh "V1 V2 ..." cmd...
L=paper_2605_10501_b200/_lib
VS=$1; shift
cp $L/libmaestro_b200.so /tmp/orig.so
for V in $VS; do
  cp $L/diag/lib_$V.so $L/libmaestro_b200.so
  echo "=== $V"
  "$@"
done
cp /tmp/orig.so $L/libmaestro_b200.so
