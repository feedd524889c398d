# Builds the sm_100a library in-tree (the .so travels to the GPU box with the repo snapshot).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude
SRC := $(wildcard paper_1602_01376_b200/csrc/*.cu)
OBJ := $(patsubst paper_1602_01376_b200/csrc/%.cu,build/%.o,$(SRC))
LIB := paper_1602_01376_b200/libinvaskit.so

all: $(LIB)

build/%.o: paper_1602_01376_b200/csrc/%.cu $(wildcard paper_1602_01376_b200/csrc/*.cuh paper_1602_01376_b200/csrc/*.h) include/invaskit.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -lcudart

clean:
	rm -rf build $(LIB)

.PHONY: all clean
