M=479168
echo "== default"; python tools/profile_knn.py --m $M --reps 3
echo "== noepi"; SG_KNN_NOEPI=1 python tools/profile_knn.py --m $M --reps 3
echo "== abl1 (no insertion)"; SG_KNN_ABL=1 python tools/profile_knn.py --m $M --reps 3
echo "== prof"; SG_LIB_PATH=$PWD/paper_2605_10135_b200/libscalegann_prof.so python tools/profile_knn.py --m $M --reps 1 --prof
echo "== ncu"; ncu --set full --import-source on --clock-control none -k regex:knn_tc -s 0 -c 1 -f -o gpurun_out/r2c_knn_full python tools/profile_knn.py --m $M --reps 1 > gpurun_out/r2c_knn_full.log 2>&1; echo ncu_rc=$?
