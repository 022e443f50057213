# graph time of n=16384 with op kinds replaced by empty kernels (timing only)
for m in 0 1 2 3 12; do
  RELAPACK_DEBUG_SKIP=$m python tools/critical_path.py 16384 U 2>&1 | head -1 | sed "s/^/skip=$m /"
done
