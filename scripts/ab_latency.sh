# batch-1 latency sweep for several builds (each copied over the in-tree lib)
cd $GRAFT_REPO_ROOT
cp paper_2604_22312_b200/libgvrtopk.so /tmp/lib_keep.so
for l in "$@"; do
  cp $l paper_2604_22312_b200/libgvrtopk.so
  echo "== $l"
  timeout 300 python scripts/latency_sweep.py --ns 8192,32768,100000,262144 --reps 20 2>&1 | python -c "
import sys, json
for line in sys.stdin:
    d = json.loads(line); print(d['N'], d['gvr']['us_median'], 'G', d['gvr_stats']['cluster'])"
done
cp /tmp/lib_keep.so paper_2604_22312_b200/libgvrtopk.so
