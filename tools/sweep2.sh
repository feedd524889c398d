for cfg in "KS_HAGER_FLUSH=64" "KS_HAGER_FLUSH=64 KS_SLAB_MAX=8" "KS_HAGER_FLUSH=128 KS_SLAB_MAX=8" "KS_HAGER_FLUSH=64 KS_SLAB_MAX=8 KS_HAGER_CTAS=64"; do
  echo "== $cfg"; env $cfg timeout 300 bash tools/bench_quick.sh 2>&1 | head -2
done
