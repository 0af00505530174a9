# Builds the in-tree C-ABI library paper_1807_06108_b200/libjmppi.so for sm_100a
# and the oracle's C helpers.  `make -j8`.
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH ?= -gencode arch=compute_100a,code=sm_100a
NVFLAGS ?= $(ARCH) -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC -Xptxas -v
PKG := paper_1807_06108_b200
SRC := $(wildcard $(PKG)/csrc/*.cu)
OBJ := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(SRC))
HDR := $(wildcard $(PKG)/csrc/*.cuh) $(PKG)/csrc/internal.h include/jmppi.h

all: $(PKG)/libjmppi.so

build/%.o: $(PKG)/csrc/%.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; exit 1)

$(PKG)/libjmppi.so: $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ)

clean:
	rm -rf build $(PKG)/libjmppi.so

.PHONY: all clean
