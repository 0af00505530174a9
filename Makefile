# Builds the in-tree C-ABI library paper_1807_06108_b200/libjmppi.so for sm_100a
# and the oracle's C helpers.  `make -j8`.
# Tuning variants: make BUILD=scratch/bX LIB=scratch/libX.so EXTRA="-DNAME=VALUE"
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH ?= -gencode arch=compute_100a,code=sm_100a
EXTRA ?=
NVFLAGS ?= $(ARCH) -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC -Xptxas -v $(EXTRA)
PKG := paper_1807_06108_b200
BUILD ?= build
LIB ?= $(PKG)/libjmppi.so
SRC := $(wildcard $(PKG)/csrc/*.cu)
OBJ := $(patsubst $(PKG)/csrc/%.cu,$(BUILD)/%.o,$(SRC))
HDR := $(wildcard $(PKG)/csrc/*.cuh) $(PKG)/csrc/internal.h include/jmppi.h

all: $(LIB)

$(BUILD)/%.o: $(PKG)/csrc/%.cu $(HDR)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(BUILD)/$*.ptxas.log || (cat $(BUILD)/$*.ptxas.log; exit 1)

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ)

clean:
	rm -rf build $(PKG)/libjmppi.so

.PHONY: all clean
