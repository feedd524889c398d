# Environment sweep of the factorization schedule: one bench_quick line per setting.
#   bash tools/sweep.sh "KS_SLAB_MAX=4" "KS_SLAB_MAX=8 KS_HAGER_CTAS=80" ...
for cfg in "$@"; do
  echo "== $cfg"; env $cfg timeout 300 bash tools/bench_quick.sh 2>&1 | head -2
done
