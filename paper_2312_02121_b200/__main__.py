"""python -m paper_2312_02121_b200 {render,gradcheck,fit} ... (cli.main)."""
import sys

from .cli import main

sys.exit(main())
