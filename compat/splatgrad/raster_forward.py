"""splatgrad.raster_forward names (sg/raster_forward.py) on the B200 build."""
from paper_2312_02121_b200.api import (ALPHA_MAX, ALPHA_MIN, SIGMA_CUT, T_MIN, ImageBuffer, PixelAux,  # noqa: F401
                                       RenderAux, RenderResult, composite_pixel, eval_alpha, render,
                                       render_brute_force)
