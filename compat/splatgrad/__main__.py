import sys

from paper_2312_02121_b200.cli import main

sys.exit(main())
