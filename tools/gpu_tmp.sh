mkdir -p gpurun_out
(python tools/probe_codec.py sc vlz --tables 4; python tools/probe_codec.py sc vlz --tables 4 --batch 8192; python tools/probe_codec.py tb vlz; python tools/probe_codec.py tb vlz --batch 65536 --tables 4; python tools/probe_codec.py sc huffman --tables 4 ) > gpurun_out/r2c.log 2>&1
cat gpurun_out/r2c.log
