# Builds paper_2407_13997_b200/libwrmg.so for sm_100a (B200).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
FLAGS := -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr -Xptxas -v
SRC := $(wildcard paper_2407_13997_b200/csrc/*.cu)
HDR := $(wildcard paper_2407_13997_b200/csrc/*.h) include/wrmg.h
OUT := paper_2407_13997_b200/libwrmg.so
OBJ := $(patsubst paper_2407_13997_b200/csrc/%.cu,build/%.o,$(SRC))

all: $(OUT)

build/%.o: paper_2407_13997_b200/csrc/%.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(ARCH) $(FLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(OUT): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -lcudart -ldl

clean:
	rm -rf build $(OUT)

.PHONY: all clean
