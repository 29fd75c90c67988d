# knn tuning sweep on one synthetic shard (m rows): plain timing per configuration
M=${M:-400000}
for cfg in "$@"; do
  echo "cfg=[$cfg] $(env $cfg SG_KNN_REPORT=1 python tools/profile_knn.py --m $M --reps 3 2>&1 | grep -v '^\[knn\]' | tail -1) fails=$(env $cfg SG_KNN_REPORT=1 python tools/profile_knn.py --m $M --reps 1 2>&1 | grep '^\[knn\]' | tail -1)"
done
