# build_var NAME "NVCC_DEFINES": stage.cu rebuilt with the given macros, linked with the
# other objects of the last `make lib` into build/var_NAME/libjanus_b200.so (A/B runs).
build_var () 
{ 
    d=build/var_$1;
    mkdir -p $d;
    /usr/local/cuda/bin/nvcc -I/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/include -Iinclude -std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr $2 -c paper_2605_18404_b200/csrc/stage.cu -o $d/stage.cu.o && objs=$(ls build/obj/*.o | grep -v stage.cu.o) && /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $d/libjanus_b200.so $d/stage.cu.o $objs -L/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/lib -l:libnccl.so.2 -Xlinker -rpath -Xlinker /opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/lib -L/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/cublas/lib -l:libcublas.so.12 -Xlinker -rpath -Xlinker /opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/cublas/lib -lcudart
}
if [ $# -gt 0 ]; then build_var "$@"; fi
