for combo in "KS_SLAB_MAX=4 KS_HAGER_CTAS=96" "KS_SLAB_MAX=8 KS_HAGER_CTAS=20" "KS_SLAB_MAX=8 KS_HAGER_CTAS=96" "KS_SLAB_MAX=4 KS_HAGER_CTAS=48" "KS_SLAB_MAX=4 KS_HAGER_CTAS=148" "KS_SLAB_MAX=8 KS_HAGER_CTAS=8"; do
  echo "[$combo]"; env $combo python tools/ablate.py 0 256 2>&1 | tail -2
done
