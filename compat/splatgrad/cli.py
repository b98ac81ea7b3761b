"""splatgrad.cli names (sg/cli.py) on the B200 build."""
from paper_2312_02121_b200.cli import main, parse_scene, read_image, serialize_scene, write_image  # noqa: F401
