# Build of the B200-native TFLA library and the CPU checkers.
#   make            -> paper_2503_14376_b200/_lib/libtfla_b200.so (sm_100a)
#   make oracle     -> oracle/_build/libtfla_oracle.so (+ oracle/_ref when /root/reference exists)
#   make hosttest   -> paper_2503_14376_b200/_lib/tfla_host_test (C++ host API smoke binary)
NVCC      ?= nvcc
CXX       ?= g++
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -ftz=true -Xcompiler -fPIC -Xptxas -v \
             -Iinclude -Ipaper_2503_14376_b200/csrc
CSRC      := paper_2503_14376_b200/csrc
OBJDIR    := build/obj
LIBDIR    := paper_2503_14376_b200/_lib
LIB       := $(LIBDIR)/libtfla_b200.so

CU_SRCS   := $(wildcard $(CSRC)/*.cu)
CPP_SRCS  := $(wildcard $(CSRC)/*.cpp)
OBJS      := $(patsubst $(CSRC)/%.cu,$(OBJDIR)/%.o,$(CU_SRCS)) \
             $(patsubst $(CSRC)/%.cpp,$(OBJDIR)/%.cpp.o,$(CPP_SRCS))
HDRS      := $(wildcard $(CSRC)/*.cuh) $(wildcard $(CSRC)/*.h) $(wildcard include/tfla/*.h) \
             $(wildcard include/tfla/*.hpp)

.PHONY: all oracle hosttest clean
all: $(LIB)

$(OBJDIR)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $@.ptxas.log || (cat $@.ptxas.log; false)

$(OBJDIR)/%.cpp.o: $(CSRC)/%.cpp $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -x cu -c $< -o $@ 2> $@.ptxas.log || (cat $@.ptxas.log; false)

$(LIB): $(OBJS)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart

hosttest: $(LIB) tests/host/tfla_host_test.cpp
	$(CXX) -O2 -std=c++17 -Iinclude -I/usr/local/cuda/include tests/host/tfla_host_test.cpp \
	    -L$(LIBDIR) -ltfla_b200 -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,'$$ORIGIN' \
	    -o $(LIBDIR)/tfla_host_test

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(LIBDIR)
	$(MAKE) -C oracle clean
