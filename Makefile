# Builds the CUDA hot path (libkkm.so, sm_100a) and the CPU oracle (liboracle.so).
PY       ?= python
NVCC     ?= nvcc
NCCL_DIR := $(shell $(PY) -c "import nvidia.nccl; print(list(nvidia.nccl.__path__)[0])")
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared --expt-relaxed-constexpr \
            -Iinclude -I$(NCCL_DIR)/include -Xptxas -warn-spills
PKG      := paper_2601_17136_b200
SRCS     := $(wildcard $(PKG)/csrc/*.cu) $(wildcard $(PKG)/csrc/*.cuh) include/kkm.h

all: $(PKG)/libkkm.so oracle/liboracle.so

$(PKG)/libkkm.so: $(SRCS)
	$(NVCC) $(NVFLAGS) $(PKG)/csrc/kkm_api.cu -o $@ -L$(NCCL_DIR)/lib -l:libnccl.so.2 \
	    -Xlinker -rpath=$(NCCL_DIR)/lib

oracle/liboracle.so: oracle/kkm_oracle.c
	gcc -O2 -fopenmp -fPIC -shared -std=c11 -fno-fast-math -ffp-contract=off $< -o $@ -lm

# A/B experiment builds: make exp NAME=x EXP="-DKKM_EXP_..." -> build/libkkm_x.so (KKM_LIBKKM selects it)
exp: $(SRCS)
	mkdir -p build
	$(NVCC) $(NVFLAGS) $(EXP) $(PKG)/csrc/kkm_api.cu -o build/libkkm_$(NAME).so -L$(NCCL_DIR)/lib -l:libnccl.so.2 \
	    -Xlinker -rpath=$(NCCL_DIR)/lib

sass: $(PKG)/libkkm.so
	cuobjdump -sass $(PKG)/libkkm.so > build_sass.txt

clean:
	rm -f $(PKG)/libkkm.so oracle/liboracle.so

.PHONY: all clean sass exp
