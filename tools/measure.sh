# Round measurement on one B200: bench line, reference arm, ncu launch list of the bench command,
# one full ncu capture of the main distance-kernel launch at the bench's largest shard size.
# Usage: bash tools/measure.sh TAG   (outputs under gpurun_out/TAG_*)
TAG=${1:-r}
mkdir -p gpurun_out
python bench.py --steps 5 --warmup 3 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?"; cat gpurun_out/${TAG}_bench.json
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err
echo "ref rc=$?"; head -c 600 gpurun_out/${TAG}_ref.json; echo
python bench.py --profile-steps --steps 1 --warmup 3 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --profile-steps --steps 1 --warmup 3 > gpurun_out/${TAG}_launches.log 2>&1
echo "launch list rc=$?"
M=${M:-479168}
python tools/profile_knn.py --m $M --reps 1 > /dev/null 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:knn_tc -s 0 -c 1 -f -o gpurun_out/${TAG}_knn_full \
    python tools/profile_knn.py --m $M --reps 1 > gpurun_out/${TAG}_knn_full.log 2>&1
echo "ncu full rc=$?"
python tools/profile_build.py --m 450000 --reps 1 > /dev/null 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"prune_kernel|reverse_merge|scatter_kernel|indeg_kernel" -c 4 -f \
    -o gpurun_out/prune_full python tools/profile_build.py --m 450000 --reps 1 > gpurun_out/${TAG}_prune_full.log 2>&1
echo "ncu prune rc=$?"
