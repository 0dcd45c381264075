"""B200-native hot path of arXiv 2202.12567: sparse sampling + low-rank completion of the
many-light lighting matrix, behind the C-ABI library liblmc.so (include/lmc.h).

    from paper_2202_12567_b200 import lmc           # loads liblmc.so (raises if missing)
    frame = lmc.Frame(scenegen.make_inputs("c2"))
    frame.run(image)        # lmc_build_slices ... lmc_resolve_image, all CUDA kernels
"""
import os

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "liblmc.so")
