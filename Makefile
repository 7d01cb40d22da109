# Builds the B200 (sm_100a) shared library and the C oracle.  `make` here
# cross-compiles without a GPU; the .so travels to the GPU box via gpurun.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 -lineinfo $(ARCH) -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
SRC := $(wildcard paper_1206_4880_b200/csrc/*.cu)
HDR := $(wildcard paper_1206_4880_b200/csrc/*.h paper_1206_4880_b200/csrc/*.cuh) include/fic_b200.h
LIB := paper_1206_4880_b200/libfic_b200.so
OBJ := $(patsubst paper_1206_4880_b200/csrc/%.cu,build/%.o,$(SRC))

all: $(LIB)

build/%.o: paper_1206_4880_b200/csrc/%.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -cudart static

clean:
	rm -rf build $(LIB)

.PHONY: all clean
