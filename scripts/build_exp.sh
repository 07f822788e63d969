# tuning builds: scripts/build_exp.sh NAME -DFLAG ...  -> paper_2507_12205_b200/exp/libNAME.so
# (use with ECSR_B200_LIB=$PWD/paper_2507_12205_b200/exp/libNAME.so)
set -e
name=$1; shift
mkdir -p paper_2507_12205_b200/exp
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2,-fopenmp,-mpopcnt "$@" \
  -shared -o paper_2507_12205_b200/exp/lib$name.so paper_2507_12205_b200/csrc/ecsr_b200.cu \
  paper_2507_12205_b200/csrc/ecsr_encoder.cpp paper_2507_12205_b200/csrc/ecsr_loader.cpp -lgomp
