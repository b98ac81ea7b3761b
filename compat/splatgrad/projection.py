"""splatgrad.projection names (sg/projection.py) on the B200 build."""
from paper_2312_02121_b200.api import DILATION, ProjectedGaussian, project_gaussian  # noqa: F401
from paper_2312_02121_b200.helpers import (bounding_radius, camera_to_pixel, project_covariance,  # noqa: F401
                                           projection_jacobian, world_to_camera)
