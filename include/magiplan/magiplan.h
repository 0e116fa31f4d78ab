/* Include-path compatibility with the reference (#include "magiplan/magiplan.h",
 * /root/reference/proj/include/magiplan/magiplan.h). */
#include "../magiplan.h"
