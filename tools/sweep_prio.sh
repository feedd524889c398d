for combo in "KS_GROUP_PRIO=0" "KS_GROUP_PRIO=1" "KS_GROUP_PRIO=1 KS_GRAPH=0" "KS_GROUP_PRIO=0 KS_GRAPH=0"; do
  echo "[$combo]"; env $combo python tools/ablate.py 0 2>&1 | tail -1
done
