# Builds the sm_100a C-ABI library in-tree: paper_2411_19588_b200/libuwsplat_b200.so
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
SRC := paper_2411_19588_b200/csrc
OBJ := build/obj
LIB := paper_2411_19588_b200/libuwsplat_b200.so
# float64 translation units that must evaluate expressions exactly like numpy
EXACT := preprocess preprocess_bwd densify backscatter
FAST := binning raster_fwd raster_bwd loss adam capi
OBJS := $(addprefix $(OBJ)/,$(addsuffix .o,$(EXACT) $(FAST)))
HDRS := $(wildcard $(SRC)/*.cuh) include/uwsplat_b200.h

all: $(LIB)

$(OBJ):
	mkdir -p $(OBJ)

$(OBJ)/preprocess.o $(OBJ)/preprocess_bwd.o $(OBJ)/densify.o $(OBJ)/backscatter.o: $(OBJ)/%.o: $(SRC)/%.cu $(HDRS) | $(OBJ)
	$(NVCC) $(NVFLAGS) -fmad=false -c $< -o $@ 2> $(OBJ)/$*.ptxas.log || (cat $(OBJ)/$*.ptxas.log; false)

$(OBJ)/%.o: $(SRC)/%.cu $(HDRS) | $(OBJ)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(OBJ)/$*.ptxas.log || (cat $(OBJ)/$*.ptxas.log; false)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS)

clean:
	rm -rf build $(LIB)

.PHONY: all clean
