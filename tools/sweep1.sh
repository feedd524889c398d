# env sweep of the factorization schedule (bench_quick per setting)
for cfg in "KS_SLAB_MAX=4" "KS_SLAB_MAX=2" "KS_SLAB_MAX=4 KS_HAGER_CTAS=52" "KS_SLAB_MAX=0" "KS_SLAB_MAX=4 KS_HAGER_SPLIT=0"; do
  echo "== $cfg"; env $cfg timeout 300 bash tools/bench_quick.sh 2>&1 | head -2
done
