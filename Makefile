# Builds the product library (paper_2204_10402_b200/libvcgpu.so, sm_100a) and the test-only
# checkers under oracle/. `python -c "import __graft_entry__ as g; g.build()"` runs this.
NVCC     ?= nvcc
HOSTCXX  ?= g++
ARCH     := -gencode arch=compute_100a,code=sm_100a
PKG      := paper_2204_10402_b200
SRC      := $(PKG)/csrc
OBJ      := build/obj
LIB      := $(PKG)/libvcgpu.so
CXXFLAGS := -O3 -std=c++17 -fPIC -fvisibility=hidden -Wall -Wextra
NVFLAGS  := -O3 -std=c++17 $(ARCH) -lineinfo -Xptxas -v -Xcompiler -fPIC,-fvisibility=hidden

CU_SRCS  := $(wildcard $(SRC)/*.cu)
CPP_SRCS := $(wildcard $(SRC)/*.cpp)
HDRS     := $(wildcard $(SRC)/*.hpp) $(wildcard $(SRC)/*.cuh) include/vcgpu.h
OBJS     := $(patsubst $(SRC)/%.cu,$(OBJ)/%.cu.o,$(CU_SRCS)) $(patsubst $(SRC)/%.cpp,$(OBJ)/%.o,$(CPP_SRCS))

CLI      := $(PKG)/bin/vcsolve

all: $(LIB) $(CLI) oracle

$(OBJ)/%.cu.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p $(OBJ)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $@.ptxas.log || (cat $@.ptxas.log; exit 1)

$(OBJ)/%.o: $(SRC)/%.cpp $(HDRS)
	@mkdir -p $(OBJ)
	$(HOSTCXX) $(CXXFLAGS) -c $< -o $@

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@.tmp $(OBJS) -Xlinker --exclude-libs,ALL -Xlinker -Bsymbolic
	mv $@.tmp $@

# the reference CLI's drop-in (tools/main.cpp), linked against the C-ABI only
$(CLI): $(PKG)/cli/vcsolve.cpp include/vcgpu.h $(LIB)
	@mkdir -p $(PKG)/bin
	$(HOSTCXX) -O2 -std=c++17 -Wall -Wextra -Iinclude $< -o $@ -L$(PKG) -lvcgpu -Wl,-rpath,'$$ORIGIN/..'

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(LIB) $(CLI)
	$(MAKE) -C oracle clean

.PHONY: all oracle clean
