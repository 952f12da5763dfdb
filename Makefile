# Native build of the sidecar data plane (sm_100a only).
#   make            libfsx.so (+ SASS/resource report in build/)
#   make oracle     checker libraries (oracle/Makefile)
NVCC ?= /usr/local/cuda/bin/nvcc
CXX ?= g++
ARCH := -gencode arch=compute_100a,code=sm_100a
PKG := paper_2603_12118_b200
CSRC := $(PKG)/csrc
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-Wall -Iinclude -I$(CSRC) \
           -Xptxas -v -cudart static
LIB := $(PKG)/libfsx.so
OBJS := build/fsx_kernels.o build/fsx_runtime.o

all: $(LIB)

build:
	mkdir -p build

build/fsx_kernels.o: $(CSRC)/fsx_kernels.cu $(CSRC)/fsx_kernels.cuh include/fsx.h | build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/fsx_kernels.ptxas.txt || { cat build/fsx_kernels.ptxas.txt; exit 1; }

build/fsx_runtime.o: $(CSRC)/fsx_runtime.cu $(CSRC)/fsx_kernels.cuh include/fsx.h | build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/fsx_runtime.ptxas.txt || { cat build/fsx_runtime.ptxas.txt; exit 1; }

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(OBJS)

oracle:
	$(MAKE) -C oracle all

# C++ fabric tests (run on the GPU by tests/test_cpp_fabric.py).
FISSIM_REF_INCLUDE ?= /root/reference/proj/include
FISSIM_REF_TESTS ?= /root/reference/proj/tests
NLOHMANN_DIR ?= /opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann
CXXTEST := $(CXX) -std=c++20 -O2 -g -rdynamic -Wall -Wno-unused-parameter -Iinclude -Itests/cpp/catch2_shim \
           -I/usr/local/cuda/include
LINKFSX := -L$(PKG) -lfsx -L/usr/local/cuda/lib64 -lcudart -lpthread \
           -Wl,-rpath,'$$ORIGIN/../$(PKG)' -Wl,-rpath,/usr/local/cuda/lib64

build/fsx_oracle_test.o: oracle/fsx_oracle.c oracle/fsx_oracle.h | build
	$(CC) -std=c11 -O2 -fPIC -c $< -o $@

build/test_fabric: tests/cpp/test_fabric.cpp tests/cpp/shim_main.cpp include/fsx/fabric.hpp \
                   build/fsx_oracle_test.o $(LIB) | build
	$(CXXTEST) -Ioracle -o $@ tests/cpp/test_fabric.cpp tests/cpp/shim_main.cpp \
	    build/fsx_oracle_test.o $(LINKFSX)

# The REFERENCE's own unit tests for the sidecar, compiled unmodified against
# the drop-in header (needs the reference tree: built here, run on the box).
build/ref_test_sidecar: $(FISSIM_REF_TESTS)/test_sidecar.cpp tests/cpp/shim_main.cpp \
                        include/fsx/fabric.hpp include/fsx/dropin/fissim/sidecar.hpp $(LIB) | build
	$(CXX) -std=c++20 -O2 -g -rdynamic -w -Iinclude/fsx/dropin -Iinclude -Itests/cpp/catch2_shim \
	    -I$(FISSIM_REF_INCLUDE) -I$(NLOHMANN_DIR) -o $@ $(FISSIM_REF_TESTS)/test_sidecar.cpp \
	    tests/cpp/shim_main.cpp $(LINKFSX)

# The reference's executor and dispatcher unit tests (encoder/LLM/talker/
# generator executors and the TaskDispatcher wired through the sidecar), also
# compiled unmodified against the drop-in.
build/ref_test_executors: $(FISSIM_REF_TESTS)/test_executor_sim.cpp $(FISSIM_REF_TESTS)/test_dispatcher.cpp \
                          tests/cpp/shim_main.cpp include/fsx/fabric.hpp \
                          include/fsx/dropin/fissim/sidecar.hpp $(LIB) | build
	$(CXX) -std=c++20 -O2 -g -rdynamic -w -Iinclude/fsx/dropin -Iinclude -Itests/cpp/catch2_shim \
	    -I$(FISSIM_REF_INCLUDE) -I$(FISSIM_REF_TESTS) -I$(NLOHMANN_DIR) -o $@ \
	    $(FISSIM_REF_TESTS)/test_executor_sim.cpp $(FISSIM_REF_TESTS)/test_dispatcher.cpp \
	    tests/cpp/shim_main.cpp $(LINKFSX)

build/dropin_criterion4: tests/cpp/dropin_criterion4.cpp include/fsx/fabric.hpp \
                         include/fsx/dropin/fissim/sidecar.hpp $(LIB) | build
	$(CXX) -std=c++20 -O2 -g -rdynamic -w -Iinclude/fsx/dropin -Iinclude -I$(FISSIM_REF_INCLUDE) -I$(NLOHMANN_DIR) \
	    -o $@ tests/cpp/dropin_criterion4.cpp $(LINKFSX)

# Multi-process executors: the worker executable and the
# REFERENCE's tests/test_worker.cpp, compiled unmodified against the drop-in
# executor_worker.hpp + sidecar.hpp.  The test reads two reference data files
# (profiles/mllm.json, apps/mllm-gemma.json) from FISSIM_REPO_ROOT; they are
# staged into build/refdata (git-ignored, travels to the GPU box with build/).
REFDATA := $(CURDIR)/build/refdata
build/fsx_worker: tests/cpp/fsx_worker_main.cpp include/fsx/dropin/fissim/executor_worker.hpp \
                  include/fsx/dropin/fissim/sidecar.hpp include/fsx/fabric.hpp $(LIB) | build
	$(CXX) -std=c++20 -O2 -g -rdynamic -w -Iinclude/fsx/dropin -Iinclude -I$(FISSIM_REF_INCLUDE) -I$(NLOHMANN_DIR) \
	    -o $@ tests/cpp/fsx_worker_main.cpp $(LINKFSX)

build/refdata: | build
	mkdir -p $(REFDATA)/tests
	cp -r $(FISSIM_REF_TESTS)/../profiles $(FISSIM_REF_TESTS)/../apps $(FISSIM_REF_TESTS)/../mixes \
	    $(FISSIM_REF_TESTS)/../clusters $(REFDATA)/
	cp -r $(FISSIM_REF_TESTS)/fixtures $(REFDATA)/tests/

# The reference's acceptance test (all 10 criteria; criterion 4 is the
# sidecar) and its control-plane unit tests, compiled unmodified against the
# drop-in headers, reading the staged reference data from build/refdata.
build/ref_acceptance: $(FISSIM_REF_TESTS)/acceptance_test.cpp build/fsx_worker \
                      include/fsx/dropin/fissim/sidecar.hpp include/fsx/dropin/fissim/executor_worker.hpp \
                      | build/refdata
	$(CXX) -std=c++20 -O2 -g -rdynamic -w -Iinclude/fsx/dropin -Iinclude -I$(FISSIM_REF_INCLUDE) -I$(NLOHMANN_DIR) \
	    -DFISSIM_REPO_ROOT='"$(REFDATA)"' -DFISSIM_CLI_BIN='"$(CURDIR)/build/fsx_worker"' \
	    -o $@ $(FISSIM_REF_TESTS)/acceptance_test.cpp $(LINKFSX)

build/ref_test_control_plane: $(FISSIM_REF_TESTS)/test_control_plane.cpp tests/cpp/shim_main.cpp \
                              build/fsx_worker include/fsx/dropin/fissim/sidecar.hpp | build/refdata
	$(CXX) -std=c++20 -O2 -g -rdynamic -w -Iinclude/fsx/dropin -Iinclude -Itests/cpp/catch2_shim \
	    -I$(FISSIM_REF_INCLUDE) -I$(FISSIM_REF_TESTS) -I$(NLOHMANN_DIR) \
	    -DFISSIM_REPO_ROOT='"$(REFDATA)"' -DFISSIM_CLI_BIN='"$(CURDIR)/build/fsx_worker"' \
	    -o $@ $(FISSIM_REF_TESTS)/test_control_plane.cpp tests/cpp/shim_main.cpp $(LINKFSX)

build/ref_test_worker: $(FISSIM_REF_TESTS)/test_worker.cpp tests/cpp/shim_main.cpp build/fsx_worker \
                       include/fsx/dropin/fissim/executor_worker.hpp | build/refdata
	$(CXX) -std=c++20 -O2 -g -rdynamic -w -Iinclude/fsx/dropin -Iinclude -Itests/cpp/catch2_shim \
	    -I$(FISSIM_REF_INCLUDE) -I$(NLOHMANN_DIR) \
	    -DFISSIM_REPO_ROOT='"$(REFDATA)"' -DFISSIM_CLI_BIN='"$(CURDIR)/build/fsx_worker"' \
	    -o $@ $(FISSIM_REF_TESTS)/test_worker.cpp tests/cpp/shim_main.cpp $(LINKFSX)

build/test_worker_ipc: tests/cpp/test_worker_ipc.cpp tests/cpp/shim_main.cpp build/fsx_worker \
                       include/fsx/dropin/fissim/executor_worker.hpp | build/refdata
	$(CXX) -std=c++20 -O2 -g -rdynamic -w -Iinclude/fsx/dropin -Iinclude -Itests/cpp/catch2_shim \
	    -I$(FISSIM_REF_INCLUDE) -I$(NLOHMANN_DIR) \
	    -DFSX_REFDATA='"$(REFDATA)"' -DFSX_WORKER_BIN='"$(CURDIR)/build/fsx_worker"' \
	    -o $@ tests/cpp/test_worker_ipc.cpp tests/cpp/shim_main.cpp $(LINKFSX)

# Whole serving experiments of the reference's bench harness against the
# drop-in (tests/cpp/app_experiment.cpp); the same file built against the
# reference's own sidecar is oracle/_ref/app_experiment_ref (oracle/Makefile).
build/app_experiment_fsx: tests/cpp/app_experiment.cpp include/fsx/fabric.hpp \
                          include/fsx/dropin/fissim/sidecar.hpp $(LIB) | build/refdata
	$(CXX) -std=c++20 -O2 -g -w -DFSX_DROPIN -Iinclude/fsx/dropin -Iinclude -I$(FISSIM_REF_INCLUDE) -I$(NLOHMANN_DIR) \
	    -DFISSIM_REPO_ROOT='"$(REFDATA)"' -DFISSIM_CLI_BIN='"$(CURDIR)/build/fsx_worker"' \
	    -o $@ tests/cpp/app_experiment.cpp $(LINKFSX)

build/ref_test_bench: $(FISSIM_REF_TESTS)/test_bench.cpp tests/cpp/shim_main.cpp \
                      include/fsx/dropin/fissim/sidecar.hpp $(LIB) | build/refdata
	$(CXX) -std=c++20 -O2 -g -rdynamic -w -Iinclude/fsx/dropin -Iinclude -Itests/cpp/catch2_shim \
	    -I$(FISSIM_REF_INCLUDE) -I$(FISSIM_REF_TESTS) -I$(NLOHMANN_DIR) \
	    -DFISSIM_REPO_ROOT='"$(REFDATA)"' -DFISSIM_CLI_BIN='"$(CURDIR)/build/fsx_worker"' \
	    -o $@ $(FISSIM_REF_TESTS)/test_bench.cpp tests/cpp/shim_main.cpp $(LINKFSX)

# Binary envelope codec: round trips against the drop-in
# envelope and its cost next to the reference JSON route.  CPU only.
build/test_envelope_codec: tests/cpp/test_envelope_codec.cpp tests/cpp/shim_main.cpp \
                           include/fsx/envelope_codec.hpp include/fsx/dropin/fissim/sidecar.hpp $(LIB) | build
	$(CXX) -std=c++20 -O2 -g -rdynamic -w -Iinclude/fsx/dropin -Iinclude -Itests/cpp/catch2_shim \
	    -I$(FISSIM_REF_INCLUDE) -I$(NLOHMANN_DIR) -o $@ tests/cpp/test_envelope_codec.cpp \
	    tests/cpp/shim_main.cpp $(LINKFSX)

# Host dg64 (fabric.hpp digest64 / digest64_par) vs the oracle restatement.  CPU only.
build/test_host_digest: tests/cpp/test_host_digest.cpp include/fsx/fabric.hpp build/fsx_oracle_test.o | build
	$(CXXTEST) -Ioracle -o $@ tests/cpp/test_host_digest.cpp build/fsx_oracle_test.o -lpthread

build/bench_pass: tests/cpp/bench_pass.cpp include/fsx/dataplane.hpp build/fsx_oracle_test.o $(LIB) | build
	$(CXXTEST) -Ioracle -o $@ tests/cpp/bench_pass.cpp build/fsx_oracle_test.o $(LINKFSX)

build/bench_fabric: tests/cpp/bench_fabric.cpp include/fsx/fabric.hpp build/fsx_oracle_test.o $(LIB) | build
	$(CXXTEST) -Ioracle -o $@ tests/cpp/bench_fabric.cpp build/fsx_oracle_test.o $(LINKFSX)

build/probe_send_phases: tests/cpp/probe_send_phases.cpp include/fsx/fabric.hpp build/fsx_oracle_test.o $(LIB) | build
	$(CXXTEST) -Ioracle -o $@ tests/cpp/probe_send_phases.cpp build/fsx_oracle_test.o $(LINKFSX)

build/probe_small_path: tests/cpp/probe_small_path.cpp include/fsx/fabric.hpp $(LIB) | build
	$(CXXTEST) -o $@ tests/cpp/probe_small_path.cpp $(LINKFSX)

# Diagnostic probes (scripts/probe_*.cu|cpp; numbers in profiles/).
build/probe_launch_floor: scripts/probe_launch_floor.cu | build
	$(NVCC) $(ARCH) -O3 -o $@ $<
build/probe_pcie_pull: scripts/probe_pcie_pull.cu | build
	$(NVCC) $(ARCH) -O3 -o $@ $<
build/probe_k1_floor: scripts/probe_k1_floor.cu build/fsx_kernels.o | build
	$(NVCC) $(ARCH) -O3 -std=c++17 -Iinclude -I$(CSRC) -o $@ $< build/fsx_kernels.o
build/probe_host_copy: scripts/probe_host_copy.cpp | build
	$(CXX) -O2 -std=c++17 -I/usr/local/cuda/include -o $@ $< -L/usr/local/cuda/lib64 -lcudart -lpthread

probes: build/probe_launch_floor build/probe_pcie_pull build/probe_k1_floor build/probe_host_copy

cpptests: probes build/test_fabric build/bench_fabric build/probe_small_path build/probe_send_phases build/bench_pass build/test_host_digest
	@if [ -f $(FISSIM_REF_TESTS)/test_sidecar.cpp ]; then \
	    $(MAKE) -s -j8 build/ref_test_sidecar build/dropin_criterion4 build/ref_test_executors \
	        build/fsx_worker build/ref_test_worker build/test_worker_ipc \
	        build/ref_acceptance build/ref_test_control_plane build/ref_test_bench \
	        build/test_envelope_codec build/app_experiment_fsx; fi

sass: $(LIB)
	/usr/local/cuda/bin/cuobjdump -sass $(LIB) > build/libfsx.sass.txt

clean:
	rm -rf build $(LIB)

.PHONY: all oracle sass clean
