# tuning builds: scripts/build_exp.sh NAME -DFLAG ...  -> build/libNAME.so (git-ignored, travels
# to the GPU box). Scripts load one by setting paper_2507_12205_b200._lib.LIB_PATH before first
# use (scripts/queue_sweep.py --lib, scripts/trace_step.py); the product never does.
# -DECSR_B200_TUNING enables the env knobs ECSR_B200_TILE/_PRE/_RECCAP/_RECMAX/_TRACE.
set -e
name=$1; shift
mkdir -p build
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2,-fopenmp,-mpopcnt "$@" \
  -shared -o build/lib$name.so paper_2507_12205_b200/csrc/ecsr_b200.cu paper_2507_12205_b200/csrc/ecsr_xchg.cu paper_2507_12205_b200/csrc/ecsr_hostio.cu \
  paper_2507_12205_b200/csrc/ecsr_encoder.cpp paper_2507_12205_b200/csrc/ecsr_loader.cpp -lgomp
