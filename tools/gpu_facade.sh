mkdir -p gpurun_out
timeout 300 tests/cpp/_build/facade_tests > gpurun_out/facade_tests.txt 2>&1; echo "facade rc=$?"
timeout 600 tests/cpp/_build/ref_conformance > gpurun_out/ref_conformance.txt 2>&1; echo "ref rc=$?"
grep "\[case\]\|summary" gpurun_out/facade_tests.txt
grep "summary" gpurun_out/ref_conformance.txt
