# Build of every native artefact (run by __graft_entry__.build()).
#   paper_1410_3060_b200/libstencil.so  -- the product: sm_100a kernels + C ABI (include/stencil.h)
#   oracle/liboracle.so                 -- TEST INFRASTRUCTURE: the CPU oracle (never linked by the product)
#   synth/libsynth.so                   -- host side of the seeded input generator
PY        ?= python
NVCC      ?= /usr/local/cuda/bin/nvcc
NCCL_INC  := $(shell $(PY) -c "import os, nvidia.nccl as m; print(os.path.join(list(m.__path__)[0], 'include'))" 2>/dev/null)
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall -Xptxas -v -I$(NCCL_INC)
CSRC      := paper_1410_3060_b200/csrc
LIB       := paper_1410_3060_b200/libstencil.so
OBJS      := build/kernels.o build/pipe.o build/pipe25.o build/runtime.o

all: $(LIB) oracle/liboracle.so synth/libsynth.so build/fp64_peak build/tmem_probe build/libenergy_probe.so

build:
	mkdir -p build

build/kernels.o: $(CSRC)/kernels.cu $(CSRC)/kernels.cuh $(CSRC)/point.cuh synth/synth.h | build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/kernels.ptxas.log || (cat build/kernels.ptxas.log; false)

build/pipe.o: $(CSRC)/pipe.cu $(CSRC)/kernels.cuh $(CSRC)/point.cuh $(CSRC)/sm100.cuh | build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/pipe.ptxas.log || (cat build/pipe.ptxas.log; false)

build/pipe25.o: $(CSRC)/pipe25.cu $(CSRC)/kernels.cuh $(CSRC)/point.cuh $(CSRC)/sm100.cuh | build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/pipe25.ptxas.log || (cat build/pipe25.ptxas.log; false)

build/runtime.o: $(CSRC)/runtime.cu $(CSRC)/kernels.cuh include/stencil.h | build
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -ldl

build/fp64_peak: tools/fp64_peak.cu | build
	$(NVCC) $(ARCH) -O3 -o $@ $<

build/tmem_probe: tools/tmem_probe.cu | build
	$(NVCC) $(ARCH) -O3 -o $@ $<

build/libenergy_probe.so: tools/energy_probe.cu | build
	$(NVCC) $(ARCH) -O3 -Xcompiler -fPIC -shared -o $@ $<

oracle/liboracle.so: oracle/oracle.c
	gcc -O2 -ffp-contract=off -fno-fast-math -fopenmp -fPIC -shared -std=c11 -o $@ $<

synth/libsynth.so: synth/synth.c synth/synth.h
	gcc -O2 -fopenmp -fPIC -shared -std=c11 -o $@ $<

clean:
	rm -rf build $(LIB) oracle/liboracle.so synth/libsynth.so

.PHONY: all clean
