# Build the sm_100a C-ABI library and the CPU oracle (test infrastructure).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -fmad=false -Xcompiler -fPIC -Xptxas -v
CSRC := paper_2310_00236_b200/csrc
LIB := paper_2310_00236_b200/lib/libhalfwave_b200.so
OBJS := $(CSRC)/build/hw_api.o $(CSRC)/build/hw_acoustic.o $(CSRC)/build/hw_elastic.o $(CSRC)/build/hw_fused2d.o $(CSRC)/build/hw_elastic2d_stream.o $(CSRC)/build/hw_acoustic3d_stream.o $(CSRC)/build/hw_tb2d.o $(CSRC)/build/hw_elastic3d_stream.o $(CSRC)/build/hw_small2d.o $(CSRC)/build/hw_acoustic3d_fused.o $(CSRC)/build/hw_acoustic3d_fused32.o $(CSRC)/build/hw_elastic2d_fused.o $(CSRC)/build/hw_elastic3d_fused.o
HDRS := $(wildcard $(CSRC)/*.cuh) $(wildcard $(CSRC)/*.h) include/halfwave_b200.h

all: $(LIB) oracle

$(CSRC)/build/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(CSRC)/build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $@.ptxas.log || (cat $@.ptxas.log; false)

$(LIB): $(OBJS)
	@mkdir -p $(dir $(LIB))
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(OBJS)

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf $(CSRC)/build $(LIB)
	$(MAKE) -C oracle clean

.PHONY: all oracle clean
