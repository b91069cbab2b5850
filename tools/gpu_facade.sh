mkdir -p gpurun_out
timeout 300 tests/cpp/_build/facade_tests > gpurun_out/facade_tests.txt 2>&1; echo "facade rc=$?"
timeout 600 tests/cpp/_build/ref_conformance > gpurun_out/ref_conformance.txt 2>&1; echo "ref rc=$?"
timeout 600 oracle/_ref/scenario_ref > gpurun_out/scen_ref.txt 2>&1; echo "scen ref rc=$?"
timeout 900 tests/cpp/_build/scenario_b200 > gpurun_out/scen_b200.txt 2>&1; echo "scen b200 rc=$?"
cmp gpurun_out/scen_ref.txt gpurun_out/scen_b200.txt && echo IDENTICAL; diff gpurun_out/scen_ref.txt gpurun_out/scen_b200.txt | head -20
grep "\[case\]\|summary" gpurun_out/facade_tests.txt
grep "summary" gpurun_out/ref_conformance.txt
