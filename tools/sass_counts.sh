#!/bin/bash
# Static SASS instruction counts of the built kernels (run here, no GPU): proof that the scan
# is tcgen05 / TMEM / bulk-copy / mbarrier code.  Output: profiles/<tag>_sass_counts.txt
TAG=${1:-r02}
LIB=paper_1802_06466_b200/_lib/librbe_cuda.so
OUT=profiles/${TAG}_sass_counts.txt
{
  echo "# cuobjdump -sass $LIB: per-kernel counts of Blackwell-specific opcodes"
  echo "# UTCIMMA = tcgen05.mma kind::i8, LDTM/STTM = tcgen05.ld/st (TMEM), UBLKCP = cp.async.bulk,"
  echo "# SYNCS = mbarrier ops, IDP = __dp4a (CUDA-core small-batch body), POPC = exact kernel"
  printf "%-70s %8s %6s %6s %7s %6s %6s %6s\n" kernel UTCIMMA LDTM STTM UBLKCP SYNCS IDP POPC
  cuobjdump -sass $LIB | awk '
    /Function :/ { if (name) print name, c1, c2, c3, c4, c5, c6, c7; name=$3; c1=c2=c3=c4=c5=c6=c7=0 }
    /UTCIMMA/ {c1++} /LDTM/ {c2++} /STTM/ {c3++} /UBLKCP/ {c4++} /SYNCS/ {c5++} /IDP/ {c6++} /POPC/ {c7++}
    END { print name, c1, c2, c3, c4, c5, c6, c7 }' | while read n a b c d e f g; do
      dn=$(echo "$n" | c++filt | sed 's/(anonymous namespace):://g; s/rbe_dev:://g' | cut -c1-70)
      printf "%-70s %8s %6s %6s %7s %6s %6s %6s\n" "$dn" $a $b $c $d $e $f $g
  done | sort
} > $OUT
echo "wrote $OUT"
