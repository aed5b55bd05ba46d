# Plain-make build of libfdl.so (same flags as paper_1711_01228_b200/_build.py) and the C example.
#   make            -> paper_1711_01228_b200/lib/libfdl.so
#   make example    -> build/layout_grid (examples/layout_grid.c against the C ABI)
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 -lineinfo -Xcompiler -fPIC,-O2,-Wall --expt-relaxed-constexpr -I include
CSRC := paper_1711_01228_b200/csrc
LIBDIR := paper_1711_01228_b200/lib
OBJS := $(LIBDIR)/fdl_sym.o $(LIBDIR)/fdl_kernels.o $(LIBDIR)/fdl_api.o
HDRS := $(CSRC)/fdl_internal.h include/fdl.h

all: $(LIBDIR)/libfdl.so

$(LIBDIR)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(ARCH) $(NVFLAGS) -c $< -o $@

$(LIBDIR)/libfdl.so: $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -cudart shared -ldl -Xlinker --no-undefined

example: $(LIBDIR)/libfdl.so
	@mkdir -p build
	gcc -O2 -Wall -I include examples/layout_grid.c -o build/layout_grid -L $(LIBDIR) -lfdl -Wl,-rpath,$(abspath $(LIBDIR)) -lm

clean:
	rm -f $(OBJS) $(LIBDIR)/libfdl.so build/layout_grid

.PHONY: all example clean
