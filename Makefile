# Build the sm_100a library and the CPU oracle (also done by __graft_entry__.build()).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v
SRC := $(wildcard paper_2101_08453_b200/csrc/*.cu)
OBJ := $(SRC:.cu=.o)

all: paper_2101_08453_b200/libwd.so oracle/liborc.so

paper_2101_08453_b200/csrc/%.o: paper_2101_08453_b200/csrc/%.cu paper_2101_08453_b200/csrc/wd_internal.cuh include/wd.h
	$(NVCC) $(NVFLAGS) -c $< -o $@

paper_2101_08453_b200/libwd.so: $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ)

oracle/liborc.so: oracle/orc.c
	gcc -O2 -ffp-contract=off -fopenmp -std=c11 -shared -fPIC -o $@ $< -lm

clean:
	rm -f $(OBJ) paper_2101_08453_b200/libwd.so oracle/liborc.so
