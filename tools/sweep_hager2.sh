for combo in "KS_HAGER_CTAS=96" "KS_HAGER_CTAS=148" "KS_HAGER_CTAS=192" "KS_HAGER_CTAS=296"; do
  echo "[$combo]"; env $combo python tools/ablate.py 0 256 2>&1 | tail -2
done
