# The GPU suite against the debug build (device-side bound checks, SG_DCHECK in csrc/), the
# substitute for compute-sanitizer, which is closed on this GPU pool.
#   SG_NVCC_FLAGS=-DSG_DEBUG_CHECKS=1 SG_OBJ_DIR=objdbg \
#     SG_LIB_PATH=$PWD/paper_2605_10135_b200/libscalegann_debug.so python -m paper_2605_10135_b200.build
#   bash tools/debug_checks.sh
SG_LIB_PATH=$PWD/paper_2605_10135_b200/libscalegann_debug.so timeout 1800 python -m pytest tests -m gpu -q -x \
    > gpurun_out/debug_checks.log 2>&1
echo "debug-checks rc=$?"; tail -3 gpurun_out/debug_checks.log
