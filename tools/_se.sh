cd $GRAFT_REPO_ROOT
for a in "1" "8 1" "8 2" "8 4" "4 2" "2 2" "2 1"; do timeout 300 python tools/shard_estimate.py $a 2>&1 | tail -1; done
