#!/bin/bash
# Bounds-checked run: the whole GPU suite against libfdehodlr_dbg.so (FDE_ASSERT enabled).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
FDE_LIB_DEBUG=1 python -c "from paper_1804_05522_b200 import _lib; print('library:', _lib.load()._name)" > gpurun_out/s21_asserts.log 2>&1
FDE_LIB_DEBUG=1 timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/s21_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s21_pytest.log
grep -c "FDE_ASSERT failed" gpurun_out/s21_pytest.log >> gpurun_out/s21_asserts.log
tail -n 4 gpurun_out/s21_pytest.log; cat gpurun_out/s21_asserts.log
