# Build every native artefact in-tree (the .so files travel to the GPU box with gpurun).
#   paper_2505_22179_b200/libw4a16.so  — the product: sm_100a kernels behind the C ABI of include/w4a16.h
#   synth/libsynth_host.so, synth/libsynth_gpu.so — seeded input generator (CPU / GPU), no method arithmetic
#   oracle/libw4a16_oracle.so          — the CPU oracle (test infrastructure; built, never linked by the product)
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -Xptxas -v
CSRC := paper_2505_22179_b200/csrc
BUILD := build/obj

LIB := paper_2505_22179_b200/libw4a16.so
OBJS := $(BUILD)/abi.o $(BUILD)/pack.o $(BUILD)/gemm_mma.o $(BUILD)/accept.o $(BUILD)/mlp_glue.o $(BUILD)/gemm_tc.o \
        $(BUILD)/lmhead.o $(BUILD)/tree_attn.o $(BUILD)/hadamard.o $(BUILD)/w4a8.o $(BUILD)/gemm_tp.o

all: $(LIB) synth/libsynth_host.so synth/libsynth_gpu.so oracle/libw4a16_oracle.so

$(BUILD):
	mkdir -p $(BUILD)

# pack.cu must not contract fp32 mul/add into FMA: its codes are bit-exact with the oracle.
$(BUILD)/pack.o: $(CSRC)/pack.cu $(CSRC)/common.cuh include/w4a16.h | $(BUILD)
	$(NVCC) $(NVFLAGS) --fmad=false -c $< -o $@ 2> $(BUILD)/pack.ptxas.txt || (cat $(BUILD)/pack.ptxas.txt; false)
$(BUILD)/%.o: $(CSRC)/%.cu $(CSRC)/common.cuh $(CSRC)/tma_host.cuh $(CSRC)/tc_ptx.cuh include/w4a16.h | $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(BUILD)/$*.ptxas.txt || (cat $(BUILD)/$*.ptxas.txt; false)

# Diagnostics build (make diag): the same library with W4A16_MMA_DIAG=1 (skip-compute / skip-load / trace
# switches of gemm_mma.cu, selected at run time by W4A16_MMA_DEBUG); loaded instead of libw4a16.so when
# W4A16_LIB=diag. Never used by tests, smoke or bench.
DIAG_LIB := paper_2505_22179_b200/libw4a16_diag.so
$(BUILD)/gemm_mma_diag.o: $(CSRC)/gemm_mma.cu $(CSRC)/common.cuh $(CSRC)/tma_host.cuh include/w4a16.h | $(BUILD)
	$(NVCC) $(NVFLAGS) -DW4A16_MMA_DIAG=1 -c $< -o $@ 2> $(BUILD)/gemm_mma_diag.ptxas.txt || (cat $(BUILD)/gemm_mma_diag.ptxas.txt; false)
$(DIAG_LIB): $(filter-out $(BUILD)/gemm_mma.o,$(OBJS)) $(BUILD)/gemm_mma_diag.o
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $^
diag: $(DIAG_LIB)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(OBJS)

synth/libsynth_host.so: synth/synth.c synth/synth.h
	gcc -O2 -fPIC -shared -ffp-contract=off -fno-fast-math -o $@ synth/synth.c
synth/libsynth_gpu.so: synth/synth_gpu.cu synth/synth.h
	$(NVCC) $(ARCH) -O3 -Xcompiler -fPIC -shared -cudart static -o $@ synth/synth_gpu.cu

oracle/libw4a16_oracle.so: oracle/w4a16_oracle.c oracle/w4a16_oracle.h
	gcc -O2 -fPIC -shared -ffp-contract=off -fno-fast-math -o $@ oracle/w4a16_oracle.c -lm -lpthread

clean:
	rm -rf build $(LIB) $(DIAG_LIB) synth/*.so oracle/*.so

.PHONY: all clean diag

# A/B variant of the mma.sync family (diagnostics): make variant V=<name> VDEFS="-DW4_MA_OC=1" builds
# libw4a16_<name>.so with gemm_mma.cu compiled under VDEFS; loaded with W4A16_LIB=<name>.
V ?= ab
VDEFS ?=
variant: $(filter-out $(BUILD)/gemm_mma.o,$(OBJS))
	$(NVCC) $(NVFLAGS) $(VDEFS) -c $(CSRC)/gemm_mma.cu -o $(BUILD)/gemm_mma_$(V).o 2> $(BUILD)/gemm_mma_$(V).ptxas.txt || (cat $(BUILD)/gemm_mma_$(V).ptxas.txt; false)
	$(NVCC) $(ARCH) -shared -cudart static -o paper_2505_22179_b200/libw4a16_$(V).so $^ $(BUILD)/gemm_mma_$(V).o
.PHONY: variant
