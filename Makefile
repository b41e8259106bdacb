# Builds libmlmcp.so (sm_100a) in-tree.  `python -c "import __graft_entry__ as g; g.build()"`
# runs the same recipe.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v
SRC := $(wildcard paper_2507_19246_b200/csrc/*.cu)
HDR := $(wildcard paper_2507_19246_b200/csrc/*.cuh) include/mlmcp.h
LIB := paper_2507_19246_b200/libmlmcp.so

CHECKED := paper_2507_19246_b200/libmlmcp_checked.so

all: $(LIB)

# device-side bounds / invariant checks (MLMCP_DCHECK), same ABI
checked: $(CHECKED)

$(CHECKED): $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -DMLMCP_CHECKED -shared -o $@ $(SRC)

$(LIB): $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRC)

clean:
	rm -f $(LIB) $(CHECKED)

.PHONY: all clean checked
