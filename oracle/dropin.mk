# The C++ drop-in layer and its reference-side checks.  Needs the reference's
# public headers (/root/reference/proj/include) — the drop-in implements
# exactly those declarations — so it is built where the reference lives
# (this container); the outputs travel to the GPU box with the snapshot.
#
#  * PRODUCT  ../paper_2401_15557_b200/libphfem_dropin.so: our
#    paper_2401_15557_b200/dropin/*.cpp, i.e. build_topology, classify_edges,
#    edge_lengths, edge_normal, red_refine, local_element_matrices,
#    assemble_* of proj/include/phfem on the B200 C ABI (libphfem_b200.so).
#    A reference build swaps proj/src/{edge_topology,refine,assembly}.cpp for
#    it.
#  * TEST INFRASTRUCTURE _ref/dropin/: the reference's own unit tests
#    (proj/tests/test_{topology,refine,assembly,parabolic}.cpp, unmodified)
#    and its remaining library TUs (mesh, sparse, parabolic, elliptic,
#    problems, quadrature, analysis; unmodified) linked against the drop-in,
#    with shim/doctest (own minimal doctest) and shim/Eigen; plus
#    libphfem_dropin_runner.so = oracle/ref_runner.cpp over the drop-in (the
#    same extern "C" surface as _ref/libphfem_ref.so, so the Python parity
#    tests can drive the drop-in like the reference).
CXX      ?= g++
REF      ?= /root/reference/proj
PKG      := ../paper_2401_15557_b200
OUT      := _ref/dropin
OBJ      := $(OUT)/obj
REFFLAGS := -std=c++20 -O3 -DNDEBUG -ffp-contract=off -fPIC -w
DIFLAGS  := -std=c++20 -O2 -fPIC -Wall -Wextra -Wno-unused-parameter
INCS     := -I../shim -I../shim/doctest -I$(REF)/include -I../include
RPATH    := -Wl,-rpath,'$$ORIGIN/../../../paper_2401_15557_b200' -Wl,-rpath,'$$ORIGIN'
DROPIN   := device edge_topology_b200 refine_b200 assembly_b200
REF_KEEP := mesh sparse parabolic elliptic problems quadrature analysis
TESTS    := test_topology test_refine test_assembly test_parabolic

DROPIN_OBJS := $(DROPIN:%=$(OBJ)/%.o)
KEEP_OBJS   := $(REF_KEEP:%=$(OBJ)/ref_%.o)
SHIMS       := $(wildcard ../shim/Eigen/*) ../shim/doctest/doctest.h

all: $(PKG)/libphfem_dropin.so $(TESTS:%=$(OUT)/%) $(OUT)/libphfem_dropin_runner.so

$(OBJ)/%.o: $(PKG)/dropin/%.cpp $(PKG)/dropin/device.hpp ../include/phfem_gpu.h $(SHIMS)
	@mkdir -p $(OBJ)
	$(CXX) $(DIFLAGS) $(INCS) -I$(PKG)/dropin -c $< -o $@

$(PKG)/libphfem_dropin.so: $(DROPIN_OBJS) $(PKG)/libphfem_b200.so
	$(CXX) -shared -o $@ $(DROPIN_OBJS) -L$(PKG) -lphfem_b200 -Wl,-rpath,'$$ORIGIN'

$(OBJ)/ref_%.o: $(REF)/src/%.cpp $(SHIMS)
	@mkdir -p $(OBJ)
	$(CXX) $(REFFLAGS) $(INCS) -c $< -o $@

$(OBJ)/t_%.o: $(REF)/tests/%.cpp $(SHIMS)
	@mkdir -p $(OBJ)
	$(CXX) $(REFFLAGS) $(INCS) -I$(REF)/tests -c $< -o $@

$(OUT)/%: $(OBJ)/t_%.o $(OBJ)/t_doctest_main.o $(KEEP_OBJS) $(PKG)/libphfem_dropin.so
	$(CXX) -o $@ $< $(OBJ)/t_doctest_main.o $(KEEP_OBJS) -L$(PKG) -lphfem_dropin -lphfem_b200 $(RPATH)

$(OBJ)/runner.o: ref_runner.cpp ../include/phfem_fields.h $(SHIMS)
	@mkdir -p $(OBJ)
	$(CXX) $(REFFLAGS) $(INCS) -c $< -o $@

$(OUT)/libphfem_dropin_runner.so: $(OBJ)/runner.o $(KEEP_OBJS) $(PKG)/libphfem_dropin.so
	$(CXX) -shared -o $@ $(OBJ)/runner.o $(KEEP_OBJS) -L$(PKG) -lphfem_dropin -lphfem_b200 $(RPATH)

.PHONY: all
.SECONDARY:
