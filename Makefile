# libprgpu (sm_100a) + CPU test infrastructure (oracle, generators).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 -lineinfo $(ARCH) -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr
CSRC := paper_2109_09527_b200/csrc
SRCS := $(CSRC)/api.cu $(CSRC)/ingest.cu $(CSRC)/preprocess.cu $(CSRC)/iterate.cu $(CSRC)/blocked.cu $(CSRC)/shard.cu $(CSRC)/multicast.cu
HDRS := $(wildcard $(CSRC)/*.cuh $(CSRC)/*.h) include/prgpu.h
LIB := paper_2109_09527_b200/libprgpu.so
OBJS := $(SRCS:.cu=.o)

all: $(LIB) oracle/liboracle.so graphgen/libgraphgen.so

$(CSRC)/%.o: $(CSRC)/%.cu $(HDRS)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -cudart static

oracle/liboracle.so: oracle/oracle.c
	gcc -O2 -ffp-contract=off -fPIC -shared -std=gnu11 -o $@ $< -lm

graphgen/libgraphgen.so: graphgen/gen.c
	gcc -O2 -fopenmp -fPIC -shared -std=gnu11 -o $@ $< -lm

clean:
	rm -f $(OBJS) $(LIB) oracle/liboracle.so graphgen/libgraphgen.so

.PHONY: all clean
