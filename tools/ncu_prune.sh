M=${1:-450000}
python tools/profile_build.py --m $M --reps 2
ncu --set full --import-source on --clock-control none -k regex:"prune|reverse" -c 4 -f -o gpurun_out/prune_full \
    python tools/profile_build.py --m $M --reps 1 > gpurun_out/prune_full.log 2>&1
tail -2 gpurun_out/prune_full.log
