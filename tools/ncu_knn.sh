# one ncu --set full capture of the main distance-kernel launch (m rows, default 200K)
M=${1:-200000}
OUT=${2:-gpurun_out/knn_full}
mkdir -p gpurun_out
python tools/profile_knn.py --m $M --reps 1 > /dev/null 2>&1 || { echo "plain run failed"; exit 1; }
ncu --set full --import-source on --clock-control none -k regex:knn_tc -s 0 -c 1 -f -o $OUT \
    python tools/profile_knn.py --m $M --reps 1 > ${OUT}.log 2>&1
tail -3 ${OUT}.log
