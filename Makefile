# Build of the janus B200 library (sm_100a only) and the oracle checkers.
#   make            -> paper_2605_18404_b200/libjanus_b200.so + oracle/_ref/*
# The .so is built in-tree (git-ignored) so it travels to the GPU box.
NVCC ?= /usr/local/cuda/bin/nvcc
CXX ?= g++
PKG := paper_2605_18404_b200
SRC := $(PKG)/csrc
OBJ := build/obj
LIB := $(PKG)/libjanus_b200.so
ARCH := -gencode arch=compute_100a,code=sm_100a
# NCCL: the torch-bundled 2.28 (same image on the GPU boxes).  Linking the
# system 2.27 would make a later `import torch` bind its libnccl.so.2 SONAME to
# 2.27 and fail (ncclDevCommCreate), which breaks torchrun launches.
NCCL_HOME ?= $(shell python -c "import nvidia.nccl as n; print(n.__path__[0])" 2>/dev/null)
# cuBLAS (generic-width path GEMMs): the torch-bundled copy too, for the same SONAME reason
CUBLAS_HOME ?= $(shell python -c "import nvidia.cublas as n; print(n.__path__[0])" 2>/dev/null)
ifneq ($(CUBLAS_HOME),)
CUBLAS_LINK := -L$(CUBLAS_HOME)/lib -l:libcublas.so.12 -Xlinker -rpath -Xlinker $(CUBLAS_HOME)/lib
else
CUBLAS_LINK := -lcublas
endif
ifneq ($(NCCL_HOME),)
NCCL_INC := -I$(NCCL_HOME)/include
NCCL_LINK := -L$(NCCL_HOME)/lib -l:libnccl.so.2 -Xlinker -rpath -Xlinker $(NCCL_HOME)/lib
else
NCCL_INC :=
NCCL_LINK := -L/usr/lib/x86_64-linux-gnu -lnccl
endif
NVFLAGS := $(NCCL_INC) -Iinclude -std=c++20 -O3 $(ARCH) -lineinfo -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
ifneq ($(TC_NT),)  # tensor-core edge kernel CTA size experiment (512 default / 1024)
OBJ := build/nt$(TC_NT)_obj
LIB := build/nt$(TC_NT)/libjanus_b200.so
NVFLAGS += -DJANUS_TC_NT=$(TC_NT)
endif
ifneq ($(FEFF_CTAS),)  # FE / FF CTAs per SM experiment
OBJ := build/feff$(FEFF_CTAS)_obj
LIB := build/feff$(FEFF_CTAS)/libjanus_b200.so
NVFLAGS += -DJANUS_FEFF_CTAS=$(FEFF_CTAS)
endif
ifeq ($(PROFILE),1)  # attribution build (JANUS_PROF_SKIP), loaded via JANUS_LIB; never the product library
OBJ := build/prof_obj
LIB := build/prof/libjanus_b200.so
NVFLAGS += -DJANUS_PROFILING
endif
ifeq ($(TRACE),1)  # phase-traced profiling build (edge_tc.cuh TC_MARK), loaded via JANUS_LIB
OBJ := build/trace_obj
LIB := build/trace/libjanus_b200.so
NVFLAGS += -DJANUS_TC_TRACE
endif
CXXFLAGS := $(NCCL_INC) -Iinclude -std=c++20 -O2 -fPIC -ffp-contract=off -Wall -Wextra -I/usr/local/cuda/include
CU_SRCS := $(wildcard $(SRC)/*.cu)
CPP_SRCS := $(wildcard $(SRC)/*.cpp)
OBJS := $(patsubst $(SRC)/%.cu,$(OBJ)/%.cu.o,$(CU_SRCS)) $(patsubst $(SRC)/%.cpp,$(OBJ)/%.cpp.o,$(CPP_SRCS))
HDRS := $(wildcard $(SRC)/*.cuh) $(wildcard $(SRC)/*.hpp) $(wildcard include/*.h) $(wildcard include/janus/*.hpp)

.PHONY: all lib oracle clean
all: lib oracle

lib: $(LIB)

$(OBJ):
	mkdir -p $(OBJ)

$(OBJ)/%.cu.o: $(SRC)/%.cu $(HDRS) | $(OBJ)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $@.ptxas.log || (cat $@.ptxas.log; exit 1)

$(OBJ)/%.cpp.o: $(SRC)/%.cpp $(HDRS) | $(OBJ)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(LIB): $(OBJS)
	mkdir -p $(dir $@)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) $(NCCL_LINK) $(CUBLAS_LINK) -lcudart

oracle:
	$(MAKE) -s -C oracle

clean:
	rm -rf build $(LIB)
	$(MAKE) -s -C oracle clean
