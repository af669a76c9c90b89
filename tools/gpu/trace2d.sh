python tools/trace_call.py annulus 3 512 512 poisson surrogate 16
python tools/trace_call.py annulus 3 512 512 poisson full
python tools/trace_call.py sinmap 3 1024 1024 biharmonic surrogate 32
