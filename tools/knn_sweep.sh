# Distance-kernel parameter sweep on one B200: each line "NAME ENV..." runs tools/profile_knn.py
# in a fresh process (the kernel reads its switches once per process); PROF=1 also runs the
# cycle-counter build.  Usage: bash tools/knn_sweep.sh CONFIG_FILE M
CFG=$1; M=${2:-479168}
while read -r name envs; do
  [ -z "$name" ] && continue
  echo "== $name ($envs)"
  env $envs python tools/profile_knn.py --m $M --reps 2 2>&1 | tail -1
  if [ -n "$PROF" ]; then
    env $envs SG_LIB_PATH=$PWD/paper_2605_10135_b200/libscalegann_prof.so python tools/profile_knn.py --m $M --reps 1 --prof 2>&1 | grep -E "warp 2:|insertions"
  fi
done < $CFG
