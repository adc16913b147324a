# TEST INFRASTRUCTURE: the reference's OWN hot-path sources, unmodified, from
# /root/reference/proj/src, compiled against the in-repo Eigen-API shim
# (Eigen 3 is absent in this image) with the reference's flags (-O3, no -march;
# -ffp-contract=off keeps x86-64 baseline rounding), plus the extern "C"
# runner.  Output: oracle/_ref/libphfem_ref.so (git-ignored; travels to the
# GPU box with the snapshot).  Never run the reference's own CMake build.
CXX      ?= g++
REF      ?= /root/reference/proj
OUT      := _ref
CXXFLAGS ?= -std=c++20 -O3 -DNDEBUG -ffp-contract=off -fPIC -w
INCS     := -I../shim -I$(REF)/include
SRCS     := mesh edge_topology refine sparse assembly parabolic elliptic analysis problems quadrature
OBJS     := $(SRCS:%=$(OUT)/%.o) $(OUT)/ref_runner.o

all: $(OUT)/libphfem_ref.so

$(OUT)/%.o: $(REF)/src/%.cpp $(wildcard ../shim/Eigen/*)
	@mkdir -p $(OUT)
	$(CXX) $(CXXFLAGS) $(INCS) -c $< -o $@

$(OUT)/ref_runner.o: ref_runner.cpp ../include/phfem_fields.h $(wildcard ../shim/Eigen/*)
	@mkdir -p $(OUT)
	$(CXX) $(CXXFLAGS) $(INCS) -c $< -o $@

$(OUT)/libphfem_ref.so: $(OBJS)
	$(CXX) -shared -Wl,-Bsymbolic -Wl,--exclude-libs,ALL -o $@ $(OBJS)

.PHONY: all
