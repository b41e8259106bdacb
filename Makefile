# Builds libmlmcp.so (sm_100a) in-tree, one object per .cu (parallel, incremental:
# `make -j8`).  `python -c "import __graft_entry__ as g; g.build()"` runs this
# Makefile.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC
SRC := $(wildcard paper_2507_19246_b200/csrc/*.cu)
HDR := $(wildcard paper_2507_19246_b200/csrc/*.cuh) include/mlmcp.h
LIB := paper_2507_19246_b200/libmlmcp.so
CHECKED := paper_2507_19246_b200/libmlmcp_checked.so
OBJ := $(patsubst paper_2507_19246_b200/csrc/%.cu,build/obj/%.o,$(SRC))
COBJ := $(patsubst paper_2507_19246_b200/csrc/%.cu,build/objc/%.o,$(SRC))

all: $(LIB)

# device-side bounds / invariant checks (MLMCP_DCHECK), same ABI
checked: $(CHECKED)

build/obj/%.o: paper_2507_19246_b200/csrc/%.cu $(HDR)
	@mkdir -p build/obj
	$(NVCC) $(NVFLAGS) -Xptxas -v -c -o $@ $< 2> build/obj/$*.ptxas.log || (cat build/obj/$*.ptxas.log; false)

build/objc/%.o: paper_2507_19246_b200/csrc/%.cu $(HDR)
	@mkdir -p build/objc
	$(NVCC) $(NVFLAGS) -DMLMCP_CHECKED -c -o $@ $<

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ)

$(CHECKED): $(COBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(COBJ)

clean:
	rm -rf build/obj build/objc $(LIB) $(CHECKED)

.PHONY: all clean checked
