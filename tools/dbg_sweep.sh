for d in 0 7 15; do echo DBG $d; VP_CONV_DBG=$d python tools/conv_density.py 2>&1 | grep "density=0.25 local=False"; done
VP_CONV_DBG=15 python tools/conv_trace.py 32 0.25 | head -8
VP_CONV_DBG=7 python tools/conv_trace.py 32 0.25 | head -8
