# Build libnmkgpu.so (sm_100a) in-tree; the .so travels to the GPU box.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
# exact IEEE arithmetic: no FMA contraction, IEEE div/sqrt, no flush-to-zero
EXACT := -fmad=false -prec-div=true -prec-sqrt=true -ftz=false
NVFLAGS := -O3 -std=c++17 $(ARCH) $(EXACT) -lineinfo -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
SRC := $(wildcard paper_1703_02438_b200/csrc/*.cu)
OBJ := $(patsubst paper_1703_02438_b200/csrc/%.cu,build/%.o,$(SRC))
LIB := paper_1703_02438_b200/libnmkgpu.so

all: $(LIB)

build/%.o: paper_1703_02438_b200/csrc/%.cu $(wildcard paper_1703_02438_b200/csrc/*.cuh) include/nmk_b200.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; exit 1)

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -lcudart_static

clean:
	rm -rf build $(LIB)

.PHONY: all clean
