# Build the B200 (sm_100a) decoder library and the host-side C helpers.
#   make            -> paper_1802_08483_b200/libbsidmap.so, oracle/libbsid_oracle.so, bsidgen/libbsidgen.so
#   make ptxas      -> register / spill report of every kernel
NVCC    ?= /usr/local/cuda/bin/nvcc
CUDA_LIB ?= /usr/local/cuda/lib64
ARCH    := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O2 --expt-relaxed-constexpr $(EXTRA)
CSRC    := paper_1802_08483_b200/csrc
OBJDIR  := build/obj
CU      := $(wildcard $(CSRC)/*.cu)
OBJS    := $(patsubst $(CSRC)/%.cu,$(OBJDIR)/%.o,$(CU))
HDRS    := $(wildcard $(CSRC)/*.cuh) include/bsidmap.h
LIB     := paper_1802_08483_b200/libbsidmap.so

all: $(LIB) oracle/libbsid_oracle.so bsidgen/libbsidgen.so examples/decode_host

$(OBJDIR)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@

# the kernel headers as C++ raw strings: the sources NVRTC compiles shapes without a unit from (jit.cu)
$(OBJDIR)/jit_sources.inc: $(wildcard $(CSRC)/*.cuh)
	@mkdir -p $(OBJDIR)
	@{ for f in $^; do printf '{"%s", R"BSIDMAPJIT(' "$$(basename $$f)"; cat $$f; printf ')BSIDMAPJIT"},\n'; done; } > $@

$(OBJDIR)/jit.o: $(CSRC)/jit.cu $(HDRS) $(OBJDIR)/jit_sources.inc
	$(NVCC) $(NVFLAGS) -I$(OBJDIR) -c $< -o $@

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart -L$(CUDA_LIB) -lnvrtc -Xlinker -rpath=$(CUDA_LIB)

oracle/libbsid_oracle.so: oracle/bsid_oracle.c
	gcc -O2 -std=c11 -fPIC -shared -fno-fast-math -ffp-contract=off -fopenmp -o $@ $< -lm

bsidgen/libbsidgen.so: bsidgen/bsidgen.c
	gcc -O2 -std=c11 -fPIC -shared -o $@ $< -lm

# the C ABI used from plain C (no Python): host-buffer decode of a small batch
examples/decode_host: examples/decode_host.c include/bsidmap.h $(LIB)
	gcc -O2 -std=c11 -Iinclude -o $@ $< -Lpaper_1802_08483_b200 -lbsidmap -Wl,-rpath,'$$ORIGIN/../paper_1802_08483_b200'

ptxas:
	@for f in $(CU); do $(NVCC) $(NVFLAGS) -Xptxas -v -c $$f -o /dev/null 2>&1 | grep -E "Compiling|registers|spill" ; done

clean:
	rm -rf build $(LIB) oracle/libbsid_oracle.so bsidgen/libbsidgen.so examples/decode_host

.PHONY: all clean ptxas
