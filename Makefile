# Builds the hbem_b200 C-ABI library for B200 (sm_100a) in-tree.
NVCC    ?= nvcc
ARCH    := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xcompiler -ffp-contract=off \
           --expt-relaxed-constexpr -Xptxas -v $(EXTRA)
CXXFLAGS:= -O3 -std=c++17 -fPIC -ffp-contract=off -Wall
SRC_DIR := paper_1711_01897_b200/csrc
BUILD   := build
LIB     := paper_1711_01897_b200/libhbem_b200.so

CU_SRCS  := $(wildcard $(SRC_DIR)/*.cu)
CPP_SRCS := $(wildcard $(SRC_DIR)/*.cpp)
OBJS     := $(patsubst $(SRC_DIR)/%.cu,$(BUILD)/%.o,$(CU_SRCS)) \
            $(patsubst $(SRC_DIR)/%.cpp,$(BUILD)/%.cpp.o,$(CPP_SRCS))
HDRS     := $(wildcard $(SRC_DIR)/*.h $(SRC_DIR)/*.cuh) include/hbem_b200.h

all: $(LIB)

$(BUILD)/%.o: $(SRC_DIR)/%.cu $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@ > $(BUILD)/$*.ptxas.log 2>&1 || (cat $(BUILD)/$*.ptxas.log; false)

$(BUILD)/%.cpp.o: $(SRC_DIR)/%.cpp $(HDRS)
	@mkdir -p $(BUILD)
	g++ $(CXXFLAGS) -I/usr/local/cuda/include -c $< -o $@

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart

clean:
	rm -rf $(BUILD) $(LIB)

.PHONY: all clean
