# build_var NAME "NVCC_DEFINES" [SOURCE]: one csrc/ source (default stage.cu)
# rebuilt with the given macros, linked with the other objects of the last
# `make lib` into build/var_NAME/libjanus_b200.so (A/B runs; tools/ab_*.sh).
build_var () {
  local d=build/var_$1 src=${3:-stage.cu}
  local site=/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia
  mkdir -p $d
  /usr/local/cuda/bin/nvcc -I$site/nccl/include -Iinclude -std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a \
    -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr $2 -c paper_2605_18404_b200/csrc/$src -o $d/$src.o &&
  local objs=$(ls build/obj/*.o | grep -v "/$src.o") &&
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $d/libjanus_b200.so $d/$src.o $objs \
    -L$site/nccl/lib -l:libnccl.so.2 -Xlinker -rpath -Xlinker $site/nccl/lib \
    -L$site/cublas/lib -l:libcublas.so.12 -Xlinker -rpath -Xlinker $site/cublas/lib -lcudart
}
if [ $# -gt 0 ]; then build_var "$@"; fi
