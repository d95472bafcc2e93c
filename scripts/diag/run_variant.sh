# Diag helper: run a command with a variant library (paper_2605_10501_b200/_lib/diag/lib_<V>.so)
# swapped in for the product library, restoring it afterwards.  Usage: run_variant.sh V cmd...
L=paper_2605_10501_b200/_lib
V=$1; shift
cp $L/libmaestro_b200.so /tmp/orig.so
cp $L/diag/lib_$V.so $L/libmaestro_b200.so
"$@"
rc=$?
cp /tmp/orig.so $L/libmaestro_b200.so
exit $rc
