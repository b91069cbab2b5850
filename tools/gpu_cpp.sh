timeout 600 python -m pytest tests -m gpu -q -k "decode_loop" > gpurun_out/cppt.txt 2>&1; tail -1 gpurun_out/cppt.txt
timeout 600 tests/cpp/_build/decode_loop
