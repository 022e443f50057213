# graph time of n=16384 with op kinds replaced by empty kernels (timing only;
# mask 1 potf2, 2 trsm, 4 gemm, 8 syrk — masks that make a pivot fail abort early)
for m in 0 1 3 12; do
  RELAPACK_DEBUG_SKIP=$m python tools/critical_path.py ${1:-16384} ${2:-U} 2>&1 | head -1 | sed "s/^/skip=$m /"
done
